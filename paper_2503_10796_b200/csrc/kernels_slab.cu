// kernels_slab.cu -- device side of the x-slab decomposition.
//
// TeraAgent partitions space into mutually exclusive volumes owned by one rank each
// (P:6058-6081); agents within the interaction distance of a border are sent to the
// neighbour as aura (halo) agents every iteration, and agents that
// leave the owned volume migrate to the authoritative rank.  Here the
// volumes are x-slabs [lo, hi) (outer slabs unbounded), one per GPU.
//   k_local_frame  exact per-axis minimum and largest diameter of this rank's agents
//                  (all-reduced by the caller into the global grid frame, R12)
//   k_classify     per agent: 1 = to the left neighbour, 2 = to the right (a bit
//                  mask for the aura: an agent near both borders goes both ways)
//   scans          order-preserving positions in the left / right lists
//   k_pack         copies the selected agents into the caller's send buffers; for a
//                  migration it also lists the leavers' slots below the new count
//   k_fill_holes   the remaining agents above the new count move into those slots:
//                  the paper's parallel removal (Fig. 5.1), O(leavers)
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

// what: BDM_PACK_MIGRATE (x < lo -> left, x >= hi -> right, moved out) or BDM_PACK_AURA
// (x < lo + margin -> left, x >= hi - margin -> right, copied).
__global__ void __launch_bounds__(256) k_classify(int64_t n, const double *__restrict__ x, double lo,
                                                  double hi, double margin, int what,
                                                  uint32_t *__restrict__ fl,
                                                  uint32_t *__restrict__ fr,
                                                  uint32_t *__restrict__ fs) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) {  // the scans run over n + 1 entries (the last gives the totals)
        fl[n] = fr[n] = 0u;
        if (fs) fs[n] = 0u;
        return;
    }
    const double px = x[i];
    uint32_t l, r;
    if (what == BDM_PACK_MIGRATE) {
        l = px < lo ? 1u : 0u;
        r = px >= hi ? 1u : 0u;
    } else {
        l = px < lo + margin ? 1u : 0u;
        r = px >= hi - margin ? 1u : 0u;
    }
    fl[i] = l;
    fr[i] = r;
    if (fs) fs[i] = (l | r) ? 0u : 1u;
}

struct PackArgs {
    int64_t n;
    bdm_agents a, L, R;
    const uint32_t *pl, *pr;  // exclusive scans (n + 1 entries)
    int what;
    uint32_t *holes;          // migration: slot of the h-th leaver below the new count
};

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

__global__ void __launch_bounds__(256) k_pack(PackArgs P, long long *__restrict__ counts,
                                              DevScalars *__restrict__ sc) {
    const int64_t nl = P.pl[P.n], nr = P.pr[P.n];
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
    const int64_t m = mig ? P.n - nl - nr : P.n;  // remaining agents
    if (i == 0) {
        counts[0] = nl;
        counts[1] = nr;
        counts[2] = m;
    }
    if (i >= P.n) return;
    const uint32_t l0 = P.pl[i], r0 = P.pr[i];
    const bool to_l = P.pl[i + 1] != l0, to_r = P.pr[i + 1] != r0;
    if (to_l) copy_agent(P.a, i, P.L, l0);
    if (to_r) copy_agent(P.a, i, P.R, r0);
    // a leaver below m leaves a hole; the leavers before i number l0 + r0
    if (mig && (to_l || to_r) && i < m) P.holes[l0 + r0] = (uint32_t)i;
}

// Remaining agents at or above m fill the holes below m in rank order (the order of
// agents in a slab never enters a result: the grid sorts them, R32).
__global__ void __launch_bounds__(256) k_fill_holes(PackArgs P) {
    const int64_t nl = P.pl[P.n], nr = P.pr[P.n];
    if (nl > P.L.capacity || nr > P.R.capacity) return;
    const int64_t m = P.n - nl - nr;
    const int64_t i = m + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    const int64_t out_i = (int64_t)(P.pl[i] + P.pr[i]);       // leavers before i
    const int64_t out_m = (int64_t)(P.pl[m] + P.pr[m]);       // leavers before m
    const bool stays = P.pl[i + 1] == P.pl[i] && P.pr[i + 1] == P.pr[i];
    if (!stays) return;
    const int64_t rank = (i - m) - (out_i - out_m);            // stayers in [m, i)
    copy_agent(P.a, i, P.a, P.holes[rank]);
}

bdm_status launch_pack_slab(Ctx *c, bdm_agents *a, double lo, double hi, double margin, int what,
                            bdm_agents *to_left, bdm_agents *to_right, long long *counts_host,
                            cudaStream_t st) {
    const int64_t n = a->n;
    {
        bdm_status s0;
        if ((s0 = need_agent_buf(c, &c->cls)) != BDM_OK) return s0;
        if ((s0 = need_agent_buf(c, &c->cls2)) != BDM_OK) return s0;
        if (what == BDM_PACK_MIGRATE && (s0 = need_agent_buf(c, &c->div_rank)) != BDM_OK)
            return s0;
    }
    uint32_t *fl = c->cls, *fr = c->cls2;
    const bool mig = what == BDM_PACK_MIGRATE;
    const unsigned nb = (unsigned)((n + 1 + 255) / 256);
    k_classify<<<nb, 256, 0, st>>>(n, a->x, lo, hi, margin, what, fl, fr, nullptr);
    BDM_LAUNCH_CHECK("k_classify");
    bdm_status s;
    if ((s = launch_scan_u32(c, fl, n + 1, st)) != BDM_OK) return s;
    if ((s = launch_scan_u32(c, fr, n + 1, st)) != BDM_OK) return s;
    PackArgs P;
    P.n = n;
    P.a = *a;
    P.L = *to_left;
    P.R = *to_right;
    P.pl = fl;
    P.pr = fr;
    P.what = what;
    P.holes = mig ? c->div_rank : nullptr;
    k_pack<<<nb, 256, 0, st>>>(P, c->pack_counts, c->sc);
    // the fill pass covers at most the n - m agents above m; launched for all n (the
    // host does not know m), its blocks past the end exit at once
    if (mig) k_fill_holes<<<nb, 256, 0, st>>>(P);
    c->launches += mig ? 3 : 2;
    BDM_LAUNCH_CHECK("k_pack");
    BDM_CUDA_TRY(cudaMemcpyAsync(counts_host, c->pack_counts, 3 * sizeof(long long),
                                 cudaMemcpyDeviceToHost, st));
    return BDM_OK;
}

}  // namespace bdm
