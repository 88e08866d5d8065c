// kernels_slab.cu -- device side of the x-slab decomposition.
//
// TeraAgent partitions space into mutually exclusive volumes owned by one rank each
// (P:6058-6081); agents within the interaction distance of a border are sent to the
// neighbour as aura (halo) agents every iteration, and agents that
// leave the owned volume migrate to the authoritative rank.  Here the
// volumes are x-slabs [lo, hi) (outer slabs unbounded), one per GPU.
//   k_local_frame  exact per-axis minimum and largest diameter of this rank's agents
//                  (all-reduced by the caller into the global grid frame, R12)
//   k_pack_count   counts the agents for the left / right neighbour (an aura agent near
//                  both borders goes both ways)
//   k_pack_copy    appends them to the caller's send buffers (warp-aggregated atomics:
//                  the order of agents never enters a result, R32) and, for a
//                  migration, lists the leavers' slots below the new count m and the
//                  stayers at or above it
//   k_pack_fill    the stayers above m move into the leavers' slots: the paper's
//                  parallel removal (Fig. 5.1), O(leavers)
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

__global__ void __launch_bounds__(256) k_local_frame(int64_t n, const double *__restrict__ x,
                                                     const double *__restrict__ y,
                                                     const double *__restrict__ z,
                                                     const double *__restrict__ d,
                                                     unsigned long long *__restrict__ enc) {
    double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, dm = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        lo0 = fmin(lo0, x[i]);
        lo1 = fmin(lo1, y[i]);
        lo2 = fmin(lo2, z[i]);
        dm = fmax(dm, d[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo0 = fmin(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
        lo1 = fmin(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
        lo2 = fmin(lo2, __shfl_xor_sync(0xffffffffu, lo2, o));
        dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&enc[0], enc_double(lo0));
        atomicMin(&enc[1], enc_double(lo1));
        atomicMin(&enc[2], enc_double(lo2));
        atomicMin(&enc[3], enc_double(-dm));  // min of -d == -(max d)
    }
}

__global__ void k_frame_init(unsigned long long *enc) {
    if (threadIdx.x < 4) enc[threadIdx.x] = enc_double(INFINITY);
}

__global__ void k_frame_decode(const unsigned long long *enc, double *out) {
    if (threadIdx.x < 4) out[threadIdx.x] = dec_double(enc[threadIdx.x]);
}

bdm_status launch_local_frame(Ctx *c, const bdm_agents *a, double *frame_dev, cudaStream_t st) {
    unsigned long long *enc = (unsigned long long *)c->pack_counts + 4;  // 4 scratch words
    k_frame_init<<<1, 32, 0, st>>>(enc);
    if (a->n > 0) {
        int64_t blocks = (a->n + 255) / 256;
        if (blocks > c->sm_count * 8) blocks = c->sm_count * 8;
        k_local_frame<<<(unsigned)blocks, 256, 0, st>>>(a->n, a->x, a->y, a->z, a->diameter, enc);
    }
    k_frame_decode<<<1, 32, 0, st>>>(enc, frame_dev);
    c->launches += 3;
    BDM_LAUNCH_CHECK("local frame");
    return BDM_OK;
}

__device__ __forceinline__ void copy_agent(const bdm_agents &s, int64_t i, const bdm_agents &d,
                                           int64_t j) {
    d.x[j] = s.x[i];
    d.y[j] = s.y[i];
    d.z[j] = s.z[i];
    d.diameter[j] = s.diameter[i];
    d.id[j] = s.id[i];
    d.flags[j] = s.flags[i];
    if (s.volume && d.volume) d.volume[j] = s.volume[i];
}

// ---- atomic-append packing (the order of a slab's agents and of its ghosts never
// enters a result: the grid sorts them, R32)
__device__ __forceinline__ void side_flags(double px, double lo, double hi, double margin, int what,
                                           bool &l, bool &r) {
    if (what == BDM_PACK_MIGRATE) {
        l = px < lo;
        r = px >= hi;
    } else {
        l = px < lo + margin;
        r = px >= hi - margin;
    }
}

// Warp-aggregated slot in a list: one atomic per warp and list.
__device__ __forceinline__ unsigned long long warp_slot(bool take, unsigned long long *ctr) {
    const unsigned b = __ballot_sync(0xffffffffu, take);
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (b && lane == __ffs(b) - 1) base = atomicAdd(ctr, (unsigned long long)__popc(b));
    base = __shfl_sync(0xffffffffu, base, b ? __ffs(b) - 1 : 0);
    return base + (unsigned long long)__popc(b & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(256) k_pack_count(int64_t n, const double *__restrict__ x,
                                                    double lo, double hi, double margin, int what,
                                                    unsigned long long *__restrict__ cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool l = false, r = false;
    if (i < n) side_flags(x[i], lo, hi, margin, what, l, r);
    const unsigned bl = __ballot_sync(0xffffffffu, l), br = __ballot_sync(0xffffffffu, r);
    if ((threadIdx.x & 31) == 0) {
        if (bl) atomicAdd(&cnt[0], (unsigned long long)__popc(bl));
        if (br) atomicAdd(&cnt[1], (unsigned long long)__popc(br));
    }
}

struct PackArgs2 {
    int64_t n;
    bdm_agents a, L, R;
    double lo, hi, margin;
    int what;
    uint32_t *holes, *fillers;  // migration: leavers below m, stayers at or above m
};

__global__ void __launch_bounds__(256) k_pack_copy(PackArgs2 P, unsigned long long *__restrict__ cnt,
                                                   long long *__restrict__ counts,
                                                   DevScalars *__restrict__ sc) {
    const int64_t nl = (int64_t)cnt[0], nr = (int64_t)cnt[1];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl > P.L.capacity || nr > P.R.capacity) {  // all-or-nothing on send capacity
        if (i == 0) {
            sc->overflow = 4;
            counts[0] = -nl;
            counts[1] = -nr;
            counts[2] = P.n;
        }
        return;
    }
    const bool mig = P.holes != nullptr;
    const int64_t m = mig ? P.n - nl - nr : P.n;
    if (i == 0) {
        counts[0] = nl;
        counts[1] = nr;
        counts[2] = m;
    }
    bool l = false, r = false;
    if (i < P.n) side_flags(P.a.x[i], P.lo, P.hi, P.margin, P.what, l, r);
    const unsigned long long jl = warp_slot(l, &cnt[2]);
    const unsigned long long jr = warp_slot(r, &cnt[3]);
    if (l) copy_agent(P.a, i, P.L, (int64_t)jl);
    if (r) copy_agent(P.a, i, P.R, (int64_t)jr);
    if (mig) {
        const bool hole = (l || r) && i < m;
        const bool filler = i < P.n && !(l || r) && i >= m;
        const unsigned long long h = warp_slot(hole, &cnt[4]);
        const unsigned long long f = warp_slot(filler, &cnt[5]);
        if (hole) P.holes[h] = (uint32_t)i;
        if (filler) P.fillers[f] = (uint32_t)i;
    }
}

__global__ void __launch_bounds__(256) k_pack_fill(PackArgs2 P, const unsigned long long *__restrict__ cnt) {
    if ((int64_t)cnt[0] > P.L.capacity || (int64_t)cnt[1] > P.R.capacity) return;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= (int64_t)cnt[4]) return;  // as many holes as fillers
    copy_agent(P.a, P.fillers[k], P.a, P.holes[k]);
}

bdm_status launch_pack_slab(Ctx *c, bdm_agents *a, double lo, double hi, double margin, int what,
                            bdm_agents *to_left, bdm_agents *to_right, long long *counts_host,
                            cudaStream_t st) {
    const int64_t n = a->n;
    const bool mig = what == BDM_PACK_MIGRATE;
    if (mig) {
        bdm_status s0;
        if ((s0 = need_agent_buf(c, &c->cls)) != BDM_OK) return s0;
        if ((s0 = need_agent_buf(c, &c->cls2)) != BDM_OK) return s0;
    }
    unsigned long long *cnt = (unsigned long long *)c->pack_counts + 8;  // 6 counters
    BDM_CUDA_TRY(cudaMemsetAsync(cnt, 0, 6 * sizeof(unsigned long long), st));
    const unsigned nb = (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1);
    k_pack_count<<<nb, 256, 0, st>>>(n, a->x, lo, hi, margin, what, cnt);
    PackArgs2 P;
    P.n = n;
    P.a = *a;
    P.L = *to_left;
    P.R = *to_right;
    P.lo = lo;
    P.hi = hi;
    P.margin = margin;
    P.what = what;
    P.holes = mig ? c->cls : nullptr;
    P.fillers = mig ? c->cls2 : nullptr;
    k_pack_copy<<<nb, 256, 0, st>>>(P, cnt, c->pack_counts, c->sc);
    if (mig) k_pack_fill<<<nb, 256, 0, st>>>(P, cnt);
    c->launches += mig ? 3 : 2;
    BDM_LAUNCH_CHECK("k_pack");
    BDM_CUDA_TRY(cudaMemcpyAsync(counts_host, c->pack_counts, 3 * sizeof(long long),
                                 cudaMemcpyDeviceToHost, st));
    return BDM_OK;
}

}  // namespace bdm
