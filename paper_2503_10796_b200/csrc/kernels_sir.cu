// kernels_sir.cu -- SIR epidemiology step.
//
// Algorithms 7-9 of the paper (algo:infection P:3220-3249, algo:recovery P:3251-3270,
// algo:random-movement P:3272-3303) on point agents in a periodic cube.  Readings
// R16-R22: infection -> recovery -> movement; neighbours from the
// start-of-step snapshot; minimum-image periodic search; literal Alg. 9 wrap; Philox
// counters (id, step, 0) and (id, step, 1).  No fused multiply-add anywhere.
//
// Only infected agents can infect, so only they are indexed (the SIR counterpart of
// the uniform grid): a hash table keyed by the fine box (edge
// L = side/D >= R) whose slots head array-based linked lists of infected agents (the
// paper's "array-based linked list"), plus a bitmap over coarse blocks of
// 16^3 fine boxes.  A query first tests the <= 8 coarse bits of its 27-box
// neighbourhood; only if one is set does it probe the 27 fine boxes.
//   k_sir_collect  snapshot of the infected agents: positions, hash insert, bitmap
//   k_sir_update   per agent, in place: infection query, recovery, movement, wrap,
//                  S/I/R counts
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

constexpr int kCoarse = 16;                  // fine boxes per coarse block (per axis)
constexpr unsigned long long kEmpty = ~0ull;
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct SirArgs {
    int64_t n;
    double *__restrict__ x;
    double *__restrict__ y;
    double *__restrict__ z;
    uint8_t *__restrict__ state;
    const uint32_t *__restrict__ id;  // nullable: id = index
    double side, L, R2, half, p_inf, p_rec;
    int D, B;                         // fine boxes / coarse blocks per axis
    uint32_t k0, k1, step;
    // infected index
    unsigned long long *__restrict__ keys;
    uint32_t *__restrict__ heads;
    uint32_t *__restrict__ next;
    double *__restrict__ ix;
    double *__restrict__ iy;
    double *__restrict__ iz;
    uint32_t *__restrict__ bitmap;
    uint32_t *__restrict__ icount;
    uint32_t icap;
    unsigned long long tmask;
    int tbits;
    unsigned long long *__restrict__ counts;  // S, I, R, new infections
};

__device__ __forceinline__ int sir_box(double v, double L, int D) {
    int b = (int)floor(v / L);
    b = b < 0 ? 0 : b;
    return b > D - 1 ? D - 1 : b;
}

__device__ __forceinline__ unsigned long long box_hash(unsigned long long key, int tbits) {
    return (key * 0x9E3779B97F4A7C15ull) >> (64 - tbits);
}

__device__ __forceinline__ double min_image(double d, double side, double half) {
    if (d > half) return d - side;
    if (d < -half) return d + side;
    return d;
}

__global__ void __launch_bounds__(256) k_sir_collect(SirArgs A, DevScalars *__restrict__ sc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n || A.state[i] != 1) return;
    const uint32_t slot = atomicAdd(A.icount, 1u);
    if (slot >= A.icap) {
        sc->overflow = 3;  // infected index too small: the update is skipped
        return;
    }
    const double px = A.x[i], py = A.y[i], pz = A.z[i];
    A.ix[slot] = px;
    A.iy[slot] = py;
    A.iz[slot] = pz;
    const int bx = sir_box(px, A.L, A.D), by = sir_box(py, A.L, A.D), bz = sir_box(pz, A.L, A.D);
    const unsigned long long key =
        ((unsigned long long)bz * A.D + (unsigned long long)by) * A.D + (unsigned long long)bx;
    unsigned long long h = box_hash(key, A.tbits);
    for (;;) {
        const unsigned long long prev = atomicCAS(&A.keys[h], kEmpty, key);
        if (prev == kEmpty || prev == key) break;
        h = (h + 1) & A.tmask;
    }
    A.next[slot] = atomicExch(&A.heads[h], slot);
    const uint32_t cb = (uint32_t)(((bz / kCoarse) * A.B + (by / kCoarse)) * A.B + (bx / kCoarse));
    atomicOr(&A.bitmap[cb >> 5], 1u << (cb & 31u));
}

// Distinct coarse blocks among those of the fine boxes b-1, b, b+1 (periodic): 1-3.
__device__ __forceinline__ int coarse_set(int b, int D, int c[3]) {
    const int lo = ((b - 1 + D) % D) / kCoarse, mid = b / kCoarse, hi = ((b + 1) % D) / kCoarse;
    int n = 0;
    c[n++] = mid;
    if (lo != mid) c[n++] = lo;
    if (hi != mid && hi != lo) c[n++] = hi;
    return n;
}

__device__ __forceinline__ bool coarse_hit(const SirArgs &A, int bx, int by, int bz) {
    int cx[3], cy[3], cz[3];
    const int nx = coarse_set(bx, A.D, cx), ny = coarse_set(by, A.D, cy), nz = coarse_set(bz, A.D, cz);
    for (int a = 0; a < nz; ++a)
        for (int b = 0; b < ny; ++b)
            for (int c = 0; c < nx; ++c) {
                const uint32_t cb = (uint32_t)((cz[a] * A.B + cy[b]) * A.B + cx[c]);
                if (A.bitmap[cb >> 5] & (1u << (cb & 31u))) return true;
            }
    return false;
}

__device__ bool infected_within(const SirArgs &A, double px, double py, double pz) {
    const int bx = sir_box(px, A.L, A.D), by = sir_box(py, A.L, A.D), bz = sir_box(pz, A.L, A.D);
    if (!coarse_hit(A, bx, by, bz)) return false;
    const int D = A.D;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int cx = (bx + dx + D) % D, cy = (by + dy + D) % D, cz = (bz + dz + D) % D;
                const unsigned long long key =
                    ((unsigned long long)cz * D + (unsigned long long)cy) * D + (unsigned long long)cx;
                unsigned long long h = box_hash(key, A.tbits);
                uint32_t head = kNone;
                for (;;) {
                    const unsigned long long k = A.keys[h];
                    if (k == kEmpty) break;
                    if (k == key) {
                        head = A.heads[h];
                        break;
                    }
                    h = (h + 1) & A.tmask;
                }
                for (uint32_t j = head; j != kNone; j = A.next[j]) {
                    const double ex = min_image(px - A.ix[j], A.side, A.half);
                    const double ey = min_image(py - A.iy[j], A.side, A.half);
                    const double ez = min_image(pz - A.iz[j], A.side, A.half);
                    const double Dd = ex * ex + ey * ey + ez * ez;
                    if (Dd <= A.R2) return true;
                }
            }
    return false;
}

__device__ __forceinline__ double wrap_alg9(double el, double max_bound) {
    el = fmod(el, max_bound);
    if (el < 0.0) el = max_bound + el;
    return el;
}

__global__ void __launch_bounds__(256) k_sir_update(SirArgs A, DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    unsigned long long cs = 0, ci = 0, cr = 0, cn = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t me = A.id ? A.id[i] : (uint32_t)i;
        const double px = A.x[i], py = A.y[i], pz = A.z[i];
        uint8_t st = A.state[i];
        const U4 w = philox10(me, 0u, A.step, 0u, A.k0, A.k1);
        // Alg. 7: infection (R17: strict '<', u = w * 2^-32)
        if (st == 0 && uniform32(w.d) < A.p_inf && infected_within(A, px, py, pz)) {
            st = 1;
            ++cn;
        }
        // Alg. 8: recovery (own state updated in sequence, R18)
        if (st == 1) {
            const U4 r = philox10(me, 0u, A.step, 1u, A.k0, A.k1);
            if (uniform32(r.a) < A.p_rec) st = 2;
        }
        A.state[i] = st;
        cs += st == 0;
        ci += st == 1;
        cr += st == 2;
        // Alg. 9: movement capped at unit length (R16), toroidal wrap (R20)
        double vx = 2.0 * uniform32(w.a) - 1.0;
        double vy = 2.0 * uniform32(w.b) - 1.0;
        double vz = 2.0 * uniform32(w.c) - 1.0;
        const double v2 = vx * vx + vy * vy + vz * vz;
        if (v2 > 1.0) {
            const double nv = sqrt(v2);
            vx = vx / nv;
            vy = vy / nv;
            vz = vz / nv;
        }
        A.x[i] = wrap_alg9(px + vx, A.side);
        A.y[i] = wrap_alg9(py + vy, A.side);
        A.z[i] = wrap_alg9(pz + vz, A.side);
    }
    // block reduction of the counters, one atomic each per block
    __shared__ unsigned long long red[4][8];
    unsigned long long v[4] = {cs, ci, cr, cn};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long t = v[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[q][wid] = t;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[threadIdx.x][k];
        if (t) atomicAdd(&A.counts[threadIdx.x], t);
    }
}

static int next_pow2_bits(int64_t v) {
    int b = 1;
    while ((1ll << b) < v) ++b;
    return b;
}

bdm_status launch_sir_step(Ctx *c, bdm_agents *a, const bdm_params *p, double side, double radius,
                           double p_inf, double p_rec, long long *counts_host, cudaStream_t st) {
    SirWs &W = c->sir;
    const int D = (int)floor(side / radius);
    if (D < 3) {
        set_error("SIR needs side / radius >= 3 boxes per axis");
        return BDM_EINVAL;
    }
    if ((long long)D * D * D >= (1ll << 62)) {
        set_error("SIR grid too large");
        return BDM_EINVAL;
    }
    const int B = (D + kCoarse - 1) / kCoarse;
    const int64_t want_icap = a->n / 16 > 65536 ? a->n / 16 : 65536;
    const int64_t icap = W.icap_override > 0 ? W.icap_override : want_icap;
    const int tbits = next_pow2_bits(2 * icap);
    const int64_t tsize = 1ll << tbits;
    const int64_t bwords = ((int64_t)B * B * B + 31) / 32;
    if (icap > W.icap || tsize > W.tsize || bwords > W.bwords) {
        BDM_CUDA_TRY(cudaStreamSynchronize(st));
        void *old[] = {W.keys, W.heads, W.next, W.ix, W.iy, W.iz, W.bitmap};
        for (void *q : old)
            if (q) cudaFree(q);
        W = SirWs{};
        if (cudaMalloc(&W.keys, tsize * 8) != cudaSuccess ||
            cudaMalloc(&W.heads, tsize * 4) != cudaSuccess ||
            cudaMalloc(&W.next, icap * 4) != cudaSuccess || cudaMalloc(&W.ix, icap * 8) != cudaSuccess ||
            cudaMalloc(&W.iy, icap * 8) != cudaSuccess || cudaMalloc(&W.iz, icap * 8) != cudaSuccess ||
            cudaMalloc(&W.bitmap, bwords * 4) != cudaSuccess ||
            (!W.misc && cudaMalloc(&W.misc, 64) != cudaSuccess)) {
            cudaGetLastError();
            set_error("SIR workspace allocation failed");
            return BDM_ECAPACITY;
        }
        W.icap = icap;
        W.tsize = tsize;
        W.bwords = bwords;
    }
    if (!W.misc) BDM_CUDA_TRY(cudaMalloc(&W.misc, 64));
    SirArgs A;
    A.n = a->n;
    A.x = a->x; A.y = a->y; A.z = a->z; A.state = a->state; A.id = a->id;
    A.side = side;
    A.L = side / (double)D;
    A.R2 = radius * radius;
    A.half = side * 0.5;
    A.p_inf = p_inf;
    A.p_rec = p_rec;
    A.D = D;
    A.B = B;
    A.k0 = (uint32_t)p->seed;
    A.k1 = (uint32_t)(p->seed >> 32);
    A.step = p->step;
    A.keys = W.keys; A.heads = W.heads; A.next = W.next;
    A.ix = W.ix; A.iy = W.iy; A.iz = W.iz;
    A.bitmap = W.bitmap;
    A.icount = (uint32_t *)W.misc;
    A.counts = (unsigned long long *)((char *)W.misc + 32);
    A.icap = (uint32_t)W.icap;
    A.tbits = tbits;
    A.tmask = (unsigned long long)(tsize - 1);
    BDM_CUDA_TRY(cudaMemsetAsync(W.keys, 0xFF, tsize * 8, st));
    BDM_CUDA_TRY(cudaMemsetAsync(W.heads, 0xFF, tsize * 4, st));
    BDM_CUDA_TRY(cudaMemsetAsync(W.bitmap, 0, ((int64_t)B * B * B + 31) / 32 * 4, st));
    BDM_CUDA_TRY(cudaMemsetAsync(W.misc, 0, 64, st));
    if (a->n > 0) {
        const unsigned nb = (unsigned)((a->n + 255) / 256);
        k_sir_collect<<<nb, 256, 0, st>>>(A, c->sc);
        int64_t ub = (a->n + 255) / 256;
        const int64_t maxb = (int64_t)c->sm_count * 16;
        if (ub > maxb) ub = maxb;
        k_sir_update<<<(unsigned)ub, 256, 0, st>>>(A, c->sc);
        c->launches += 2;
        BDM_LAUNCH_CHECK("SIR kernels");
    }
    if (counts_host)
        BDM_CUDA_TRY(cudaMemcpyAsync(counts_host, A.counts, 4 * sizeof(long long),
                                     cudaMemcpyDeviceToHost, st));
    return BDM_OK;
}

}  // namespace bdm
