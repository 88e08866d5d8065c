// bdm_internal.cuh -- shared declarations of the sm_100a implementation of bdm.h.
//
// Device helpers (Philox, ordered double encoding, blocked-Morton key) and the
// library context.  Nothing here is shared with oracle/ (the CPU oracle has its own
// independent implementation of every formula).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <unordered_set>

#include "bdm.h"

namespace bdm {

// ------------------------------------------------------------------ error plumbing
void set_error(const std::string &msg);
bdm_status cuda_fail(cudaError_t e, const char *what);

#define BDM_CUDA_TRY(expr)                                              \
    do {                                                                \
        cudaError_t e__ = (expr);                                       \
        if (e__ != cudaSuccess) return ::bdm::cuda_fail(e__, #expr);    \
    } while (0)

#define BDM_LAUNCH_CHECK(what)                                          \
    do {                                                                \
        cudaError_t e__ = cudaGetLastError();                           \
        if (e__ != cudaSuccess) return ::bdm::cuda_fail(e__, what);     \
    } while (0)

// ------------------------------------------------------------------ device scalars
// Written and read only by kernels (no host round trip inside a step).
struct DevScalars {
    unsigned long long enc_lo[3], enc_hi[3], enc_dmax;  // ordered encodings (atomics)
    double R, R2, L;
    double o[3], hi[3];
    int32_t dims[3];
    int32_t T[3];          // tiles per axis = ceil(dims / 4) (a multiple of 8 in Hilbert order)
    long long nslots;      // T0*T1*T2*64
    long long slot_cap;    // allocated slots (host-written)
    int32_t overflow;      // latched: nslots > slot_cap
    int32_t nonfinite;     // latched: a position was NaN/Inf
    unsigned long long stats[5];  // cand, nbr, cont, n_static, n_moved
    int32_t boff[3];       // lattice offset: box index = floor((x - o)/L) - boff (R12, 8(e))
    int32_t has_frame;     // the origin came from a global frame (multi-GPU)
    unsigned int n_dense;  // dense tiles handed from the tile kernel to the dense kernel
    unsigned int dense_next;  // dense kernel work counter (box tasks taken)
    unsigned int tile_next;   // tile kernel work counter (tiles taken)
    uint32_t scan_epoch;      // tag of the slot scan's look-back words (k_zero_counts bumps
                              // it on the device, so graph replays get fresh tags)
    double torus_side;        // > 0: the grid is the toroidal lattice of [0, side)^3 (R52)
    double dmax_prev;      // max diameter of the grid build's input (the step keeps it)
    int32_t tile_order;    // option "tile_order" (row f1): 0 row-major tiles, 1 blocked Hilbert
    uint16_t hilb[512];    // blocked Hilbert: local tile (x | y<<3 | z<<6) -> curve position
    uint16_t hilb_inv[512];  // curve position -> local tile
};

struct Dist;  // x-slab exchange state (dist_abi.cu)

// SIR workspace (kernels_sir.cu), allocated on first use
struct SirWs {
    unsigned long long *keys = nullptr;
    unsigned long long *heads = nullptr;
    uint32_t *next = nullptr, *bitmap = nullptr;
    unsigned long long stamp = 0;
    double *ix = nullptr, *iy = nullptr, *iz = nullptr;
    void *misc = nullptr;   // infected count + 4 counters
    int64_t icap = 0, tsize = 0, bwords = 0;
    int64_t icap_override = 0;
};

// Aura codec workspace (kernels_aura.cu, row f3), allocated on first use
struct AuraWs {
    uint32_t *u32a = nullptr, *u32b = nullptr;
    int64_t u32a_cap = 0, u32b_cap = 0;
    uint8_t *pay = nullptr, *tmp = nullptr;
    int64_t pay_cap = 0, tmp_cap = 0;
    uint32_t *sizes = nullptr;
    int64_t sizes_cap = 0;
    int *err = nullptr;
    long long *res = nullptr;
};

// Agents per box at or below which two-tile units (tile_depth 2) are used in auto mode: a
// unit's region then holds 360 boxes x 1.0 = 360 agents on average, 3 sd under the
// 416-agent staging limit.
constexpr double kSparseDensity = 1.0;

// Kernel attributes and occupancy are set once per device (arrays indexed by device).
constexpr int kMaxDevices = 64;

// ------------------------------------------------------------------ library context
struct Ctx {
    int device = 0;
    int sm_count = 148;
    int64_t agent_cap = 0;
    int64_t slot_cap = 0;
    // per-agent workspace
    uint32_t *key = nullptr, *rank = nullptr;          // unsorted order
    uint32_t *perm_tmp = nullptr, *skey = nullptr, *sid = nullptr;  // after scatter
    double *sx = nullptr, *sy = nullptr, *sz = nullptr, *sd = nullptr;  // sorted SoA
    uint32_t *sidf = nullptr, *sflags = nullptr;
    // allocated on first use (need_agent_buf), so the mechanics path alone holds
    // 60 B/agent of workspace (cfg5 on one GPU)
    double *svol = nullptr;                            // sorted volume (when present)
    uint32_t *div_rank = nullptr;                      // growth/division: flag -> rank by id
    long long *n_new = nullptr;                        // growth/division: new agent count
    // grid
    uint32_t *box_start = nullptr;  // slot_cap + 1
    uint32_t *dense_list = nullptr; // 2 (slot_cap / 64) + 2 half-tile entries (dense regions)
    uint32_t *dense_scr = nullptr;  // dense kernel: per-warp octant-order scratch
    int64_t dense_scr_cap = 0;
    uint32_t *onco_id = nullptr;    // row f2: divider flags by id, then their ranks
    int64_t onco_id_cap = 0;
    long long *onco_out = nullptr;  // row f2: new n, new id_next
    uint32_t *block_sums = nullptr;
    int64_t block_sums_cap = 0;
    unsigned long long *scan_state = nullptr;  // single-pass slot scan: per-tile look-back words
    int64_t scan_state_cap = 0;
    double torus_side = 0.0;   // bdm_step with boundary 2 builds the grid on this torus (R52)
    double grid_torus = 0.0;   // the torus side the current grid was built on (0: none)
    // misc
    unsigned long long *pair_count = nullptr;
    DevScalars *sc = nullptr;       // device
    DevScalars *sc_host = nullptr;  // pinned mirror
    // bookkeeping: the grid of the last bdm_grid_build
    bool grid_valid = false;
    const double *grid_x = nullptr;
    int64_t grid_n = 0;
    int64_t grid_ng = 0;               // ghosts in the last grid build
    uint32_t *lrank = nullptr;         // sorted slot -> output index of local agents
    const double *frame = nullptr;     // device: global (o[3], -dmax) or NULL (local frame)
    uint32_t *cls = nullptr;           // slab packing: per-agent class / scan scratch
    uint32_t *cls2 = nullptr;
    long long *pack_counts = nullptr;  // device: left, right, remaining
    int64_t launches = 0;  // kernels launched (host-side count)
    int mech_kernel = 5;   // option "mech_kernel": 5 tile7 (default), 0 tile6, 1 per-agent reference, 2-4 variants
    int prefilter = 1;     // option "prefilter": fp32 conservative candidate test in the tile kernel
    int fuse_reduce = 0;   // option "fuse_reduce": next step's a1 extent from the mech epilogue
    int dense = 1;         // option "dense": dense regions go to the dense-box kernel
    int tile_depth = 0;    // option "tile_depth": 0 auto (by agents per box), 1, 2 (two-tile units)
    double density_hint = 0.0;  // agents per box of the first grid build (auto depth)
    int32_t *dims_hint = nullptr;  // pinned: box counts of a recent grid build (auto depth)
    int64_t hint_n = 0;            // agents of the build whose counts are in flight
    cudaEvent_t hint_ev = nullptr; // recorded after the dims_hint copy
    bool hint_pending = false;     // a copy is in flight: dims_hint is not to be read yet
    double hint_density = 0.0;     // agents per box of the last completed copy
    int diffuse_tma = 1;   // option "diffuse_tma": TMA-pipelined stencil when nx is even
    int tile_order = 0;    // option "tile_order" (row f1): 0 row-major, 1 blocked Hilbert
    int64_t sort_every = 1;  // option "sort_every" (row f1): reorder the caller's SoA every K-th build
    int64_t grid_builds = 0;
    bool keep_order = false;  // this grid's mechanics writes back in the input order (via perm)
    uint32_t *perm = nullptr; // sorted slot -> input index (optional, sort_every != 1)
    bool fused_valid = false;          // the scalars hold the extent of (fused_x, fused_n)
    const double *fused_x = nullptr;
    int64_t fused_n = 0;
    SirWs sir;
    AuraWs aura;
    Dist *dist = nullptr;  // bdm_dist_init / bdm_dist_init_virtual
    // bdm_create_ex: the caller's allocator for the per-agent, grid and exchange buffers
    // (NULL: cudaMalloc / cudaFree), and the blocks it handed out
    bdm_alloc_fn alloc_fn = nullptr;
    bdm_free_fn free_fn = nullptr;
    void *alloc_ctx = nullptr;
    std::unordered_set<void *> user_blocks;
    int64_t max_ghosts = 0;
};

// Library-owned device memory of the step path: through the caller's allocator when
// bdm_create_ex was given one, else cudaMalloc / cudaFree.  Called at creation and capacity
// growth (after a device synchronization; stream NULL) and when an exchange buffer grows
// (after the exchange's host synchronization, with the exchange's stream), never inside a
// step of steady size.
inline cudaError_t ctx_malloc(Ctx *c, void **p, size_t bytes, cudaStream_t st = nullptr) {
    if (c && c->alloc_fn) {
        void *q = c->alloc_fn(bytes ? bytes : 1, (void *)st, c->alloc_ctx);
        if (!q) {
            *p = nullptr;
            return cudaErrorMemoryAllocation;
        }
        c->user_blocks.insert(q);
        *p = q;
        return cudaSuccess;
    }
    return cudaMalloc(p, bytes ? bytes : 1);
}
inline void ctx_free(Ctx *c, void *p) {
    if (!p) return;
    if (c && c->free_fn && c->user_blocks.erase(p)) {
        c->free_fn(p, nullptr, c->alloc_ctx);
        return;
    }
    cudaFree(p);
}

// An optional per-agent buffer (agent_cap + 1 entries), allocated on first use.
template <class T>
inline bdm_status need_agent_buf(Ctx *c, T **p) {
    if (*p) return BDM_OK;
    const cudaError_t e = ctx_malloc(c, (void **)p, (size_t)(c->agent_cap + 1) * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return cuda_fail(e, "allocation of an optional per-agent buffer");
    }
    return BDM_OK;
}

// ------------------------------------------------------------------ device helpers
__device__ inline unsigned long long enc_double(double v) {
    // monotone map double -> u64 (for atomicMin/atomicMax on doubles)
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ inline double dec_double(unsigned long long e) {
    unsigned long long b = (e & 0x8000000000000000ull) ? (e & 0x7FFFFFFFFFFFFFFFull) : ~e;
    return __longlong_as_double((long long)b);
}

// Philox4x32-10 (Salmon et al. SC'11), the counter-based generator the paper
// proposes for order-independent per-agent randomness.
struct U4 {
    uint32_t a, b, c, d;
};
__device__ inline U4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                              uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return U4{c0, c1, c2, c3};
}
// 53-bit uniform in [0,1) from two words (R29): ((a>>5)*2^26 + (b>>6)) * 2^-53.
__device__ inline double uniform53(uint32_t a, uint32_t b) {
    return (double)(((unsigned long long)(a >> 5) << 26) | (unsigned long long)(b >> 6)) *
           0x1p-53;
}
__device__ inline double uniform32(uint32_t w) { return (double)w * 0x1p-32; }

// Tile numbering (R32, row f1).  Row-major: (tz*T1 + ty)*T0 + tx.  Blocked Hilbert
// (hilb != NULL, T0 and T1 multiples of 8): super-tiles of 8^3 tiles numbered row-major,
// the 512 tiles inside a super-tile along a 3-D Hilbert curve (table in DevScalars).
__device__ __forceinline__ uint32_t tile_rank(int tx, int ty, int tz, int T0, int T1,
                                              const uint16_t *hilb) {
    if (!hilb) return (uint32_t)((tz * T1 + ty) * T0 + tx);
    const uint32_t sup = (uint32_t)(((tz >> 3) * (T1 >> 3) + (ty >> 3)) * (T0 >> 3) + (tx >> 3));
    return sup * 512u + hilb[((tz & 7) << 6) | ((ty & 7) << 3) | (tx & 7)];
}
// inverse of tile_rank
__device__ __forceinline__ void tile_xyz(uint32_t t, int T0, int T1, const uint16_t *hilb_inv,
                                         int &tx, int &ty, int &tz) {
    if (!hilb_inv) {
        tx = (int)(t % (uint32_t)T0);
        ty = (int)((t / (uint32_t)T0) % (uint32_t)T1);
        tz = (int)(t / ((uint32_t)T0 * (uint32_t)T1));
        return;
    }
    const uint32_t sup = t >> 9, h = hilb_inv[t & 511u];
    const uint32_t S0 = (uint32_t)T0 >> 3, S1 = (uint32_t)T1 >> 3;
    tx = (int)((sup % S0) * 8u + (h & 7u));
    ty = (int)(((sup / S0) % S1) * 8u + ((h >> 3) & 7u));
    tz = (int)((sup / (S0 * S1)) * 8u + (h >> 6));
}

// Slot of box (bx, by, bz): tile number * 64 + the 6-bit Morton code inside the 4x4x4
// tile, x in the lowest bit.
__device__ __forceinline__ uint32_t box_key(int bx, int by, int bz, int T0, int T1,
                                            const uint16_t *hilb = nullptr) {
    const uint32_t tile = tile_rank(bx >> 2, by >> 2, bz >> 2, T0, T1, hilb);
    const uint32_t m = (uint32_t)((bx & 1) | ((by & 1) << 1) | ((bz & 1) << 2) |
                                  ((bx & 2) << 2) | ((by & 2) << 3) | ((bz & 2) << 4));
    return tile * 64u + m;
}
__device__ __forceinline__ const uint16_t *sc_hilb(const DevScalars *sc) {
    return sc->tile_order ? sc->hilb : nullptr;
}
__device__ __forceinline__ const uint16_t *sc_hilb_inv(const DevScalars *sc) {
    return sc->tile_order ? sc->hilb_inv : nullptr;
}

// R28: deterministic cube root.  v = m 2^e (frexp, m in [0.5, 1)); y0 = 2^k with
// k = floor((e+1)/3); exactly 8 Newton steps y <- (2y + v/(y*y))/3 without fma
// (the library is compiled with -fmad=false).
__device__ __forceinline__ double cbrt_det(double v) {
    if (!(v > 0.0)) return 0.0;
    int e;
    (void)frexp(v, &e);
    const int num = e + 1;
    const int k = num >= 0 ? num / 3 : -((-num + 2) / 3);
    double y = ldexp(1.0, k);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const double yy = y * y;
        const double q = v / yy;
        const double t = 2.0 * y + q;
        y = t / 3.0;
    }
    return y;
}

// R13: axis uniform on the sphere by rejection in the unit ball; try k uses Philox
// counter (id_lo, id_hi, step, 3 + 4k); after 16 rejections the axis is +x.
__device__ __forceinline__ void division_axis(uint32_t k0, uint32_t k1, uint32_t id,
                                              uint32_t step, double &ux, double &uy,
                                              double &uz) {
    for (uint32_t k = 0; k < 16; ++k) {
        const U4 w = philox10(id, 0u, step, 3u + 4u * k, k0, k1);
        const double vx = 2.0 * uniform32(w.a) - 1.0;
        const double vy = 2.0 * uniform32(w.b) - 1.0;
        const double vz = 2.0 * uniform32(w.c) - 1.0;
        const double n2 = vx * vx + vy * vy + vz * vz;
        if (n2 > 0.0 && n2 <= 1.0) {
            const double nn = sqrt(n2);
            ux = vx / nn;
            uy = vy / nn;
            uz = vz / nn;
            return;
        }
    }
    ux = 1.0;
    uy = 0.0;
    uz = 0.0;
}

constexpr uint32_t kChanged = BDM_FLAG_MOVED | BDM_FLAG_GREW | BDM_FLAG_ADDED;
constexpr uint32_t kGhost = 1u << 31;  // internal sorted-workspace flag: aura (ghost) agent

// ------------------------------------------------------------------ launchers
// grid (kernels_grid.cu)
bdm_status launch_init_spheres(const bdm_agents *a, int64_t id0, int64_t n, uint64_t seed,
                               double side, double d_lo, double d_width, int d_random,
                               cudaStream_t st);
bdm_status launch_grid_geometry(Ctx *c, const bdm_agents *a, const bdm_agents *g, double radius,
                                cudaStream_t st);
bdm_status launch_grid_sort(Ctx *c, const bdm_agents *a, const bdm_agents *g, cudaStream_t st);
// slabs (kernels_slab.cu)
bdm_status launch_local_frame(Ctx *c, const bdm_agents *a, double *frame_dev, cudaStream_t st);
bdm_status launch_pack_slab(Ctx *c, bdm_agents *a, double lo, double hi, double margin, int what,
                            bdm_agents *to_left, bdm_agents *to_right, long long *counts_host,
                            cudaStream_t st);
// mechanics (kernels_mech.cu)
bdm_status launch_mech(Ctx *c, bdm_agents *a, const bdm_params *p, cudaStream_t st);
bdm_status launch_pairs(Ctx *c, int64_t n, uint64_t *pairs, int64_t cap, cudaStream_t st);
bdm_status launch_peak_dfma(int sm_count, double *dfma_per_s);
bdm_status launch_selftest_recip_div(Ctx *c, int64_t n, uint64_t seed, unsigned long long *mismatches);
// generic exclusive scan of m u32 values in place (kernels_grid.cu)
bdm_status launch_scan_u32(Ctx *c, uint32_t *data, long long m, cudaStream_t st);
int64_t scan_block_count(int64_t m);
// oncology behaviour + removal (kernels_onco.cu)
bdm_status launch_onco_step(Ctx *c, bdm_agents *a, uint32_t *age, int64_t age_cap,
                            const bdm_onco_params *p, int64_t id_next, long long *out_host,
                            cudaStream_t st);
// delta + LZ4 aura codec (kernels_aura.cu)
int64_t aura_max_size(int64_t nref, int64_t n);
bdm_status launch_aura_reference(Ctx *c, const bdm_agents *m, bdm_agents *r, cudaStream_t st);
bdm_status launch_aura_encode(Ctx *c, const bdm_agents *m, const bdm_agents *r, uint8_t *out,
                              int64_t out_cap, int64_t *out_size, cudaStream_t st);
bdm_status launch_aura_decode(Ctx *c, const uint8_t *in, int64_t in_size, const bdm_agents *r,
                              bdm_agents *m, cudaStream_t st);
void free_aura(Ctx *c);
// x-slab exchange (dist_abi.cu)
void free_dist(Ctx *c);
// SIR (kernels_sir.cu)
bdm_status launch_sir_step(Ctx *c, bdm_agents *a, const bdm_params *p, double side, double radius,
                           double p_inf, double p_rec, long long *counts_host, cudaStream_t st);
// diffusion, secretion, chemotaxis (kernels_diffusion.cu)
bdm_status launch_diffuse(Ctx *c, const double *u_in, double *u_out, const bdm_grid3 *g,
                          double nu, double mu, double dt, cudaStream_t st);
bdm_status launch_secrete(Ctx *c, const bdm_agents *a, const uint8_t *type, int type_sel, double q,
                          double *u, const bdm_grid3 *g, cudaStream_t st);
bdm_status launch_chemotaxis(Ctx *c, bdm_agents *a, const uint8_t *type, int type_sel,
                             double weight, const double *u, const bdm_grid3 *g, cudaStream_t st);
// growth + division (kernels_divide.cu)
bdm_status launch_grow_divide(Ctx *c, bdm_agents *a, double growth, double v_max, double vol_to_r3,
                              uint64_t seed, uint32_t step, long long *n_new_host, cudaStream_t st);

}  // namespace bdm
