// kernels_grid.cu -- population init and the uniform-grid build.
//
//   a1  k_reduce + k_setup        exact per-axis min/max and max diameter, then
//                                 R, L = R(1+2^-20), origin, dims, tiles, nslots
//   a2  k_key                     box -> blocked-Morton slot, atomic per-slot rank
//   a3  k_scan_*                  exclusive scan of slot counts -> box_start
//   a4  k_scatter + k_fix_gather  counting-sort scatter, ascending-id order inside
//                                 a box, gather of the SoA into the sorted workspace
//
// Paper: "Environment Search" P:2584-2598; sec:grid P:4487-4530 (boxes, 27-box
// search, array-based linked list); sec:load-balancing P:4720-4838 (Morton order,
// prefix sum over boxes P:4820-4827, copy to the new position P:4829-4835).
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

// ============================================================== population init
__global__ void k_init_spheres(int64_t id0, int64_t n, uint32_t k0, uint32_t k1, double side,
                               double d_lo, double d_width, int d_random, double *__restrict__ x,
                               double *__restrict__ y, double *__restrict__ z,
                               double *__restrict__ d, uint32_t *__restrict__ id,
                               uint32_t *__restrict__ flags) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long a = (unsigned long long)(id0 + k);
        const uint32_t lo = (uint32_t)a, hi = (uint32_t)(a >> 32);
        const U4 w = philox10(lo, hi, 0xFFFFFFFFu, 2u, k0, k1);
        x[k] = uniform53(w.a, w.b) * side;
        y[k] = uniform53(w.c, w.d) * side;
        const U4 v = philox10(lo, hi, 0xFFFFFFFEu, 2u, k0, k1);
        z[k] = uniform53(v.a, v.b) * side;
        if (d_random) {
            const U4 u = philox10(lo, hi, 0xFFFFFFFDu, 2u, k0, k1);
            d[k] = d_lo + d_width * uniform53(u.a, u.b);
        } else {
            d[k] = d_lo;
        }
        id[k] = (uint32_t)a;
        flags[k] = BDM_FLAG_ADDED;
    }
}

bdm_status launch_init_spheres(const bdm_agents *a, int64_t id0, int64_t n, uint64_t seed,
                               double side, double d_lo, double d_width, int d_random,
                               cudaStream_t st) {
    if (n == 0) return BDM_OK;
    const int threads = 256;
    const int64_t blocks = (n + threads - 1) / threads;
    k_init_spheres<<<(unsigned)(blocks < 1184 * 16 ? blocks : 1184 * 16), threads, 0, st>>>(
        id0, n, (uint32_t)seed, (uint32_t)(seed >> 32), side, d_lo, d_width, d_random, a->x,
        a->y, a->z, a->diameter, a->id, a->flags);
    BDM_LAUNCH_CHECK("k_init_spheres");
    return BDM_OK;
}

// ============================================================== a1: global scalars
__global__ void k_reset_scalars(DevScalars *sc) {
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            sc->enc_lo[a] = enc_double(INFINITY);
            sc->enc_hi[a] = enc_double(-INFINITY);
        }
        sc->enc_dmax = enc_double(-INFINITY);
    }
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Exact min/max (comparisons only): per-thread, warp shuffles, shared memory, one
// atomic per block on the ordered encodings.
__global__ void __launch_bounds__(256) k_reduce(int64_t n, const double *__restrict__ x,
                                                const double *__restrict__ y,
                                                const double *__restrict__ z,
                                                const double *__restrict__ d, DevScalars *sc) {
    double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY;
    double hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY, dm = -INFINITY;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double px = x[i], py = y[i], pz = z[i], pd = d[i];
        bad |= !isfinite(px) || !isfinite(py) || !isfinite(pz) || !isfinite(pd);
        lo0 = fmin(lo0, px); hi0 = fmax(hi0, px);
        lo1 = fmin(lo1, py); hi1 = fmax(hi1, py);
        lo2 = fmin(lo2, pz); hi2 = fmax(hi2, pz);
        dm = fmax(dm, pd);
    }
    lo0 = warp_min(lo0); lo1 = warp_min(lo1); lo2 = warp_min(lo2);
    hi0 = warp_max(hi0); hi1 = warp_max(hi1); hi2 = warp_max(hi2); dm = warp_max(dm);
    __shared__ double sh[8][7];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[w][0] = lo0; sh[w][1] = lo1; sh[w][2] = lo2;
        sh[w][3] = hi0; sh[w][4] = hi1; sh[w][5] = hi2; sh[w][6] = dm;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&sc->nonfinite, 1);
    if (threadIdx.x < 7) {
        const int q = threadIdx.x;
        double v = sh[0][q];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            v = q < 3 ? fmin(v, sh[k][q]) : fmax(v, sh[k][q]);
        const unsigned long long e = enc_double(v);
        if (q < 3) atomicMin(&sc->enc_lo[q], e);
        else if (q < 6) atomicMax(&sc->enc_hi[q - 3], e);
        else atomicMax(&sc->enc_dmax, e);
    }
}

// R, L, origin, dims, tiles, slot count; latches overflow if the slots do not fit.
// With a global frame (multi-GPU, 8(e)) the origin and R come from the frame (the
// all-reduced minimum corner and largest diameter of every rank) and the local
// extent only fixes the lattice offset and dims.
__global__ void k_setup(DevScalars *sc, double radius, const double *__restrict__ frame,
                        int reset_after, double torus_side) {
    if (threadIdx.x != 0) return;
    const double R = radius > 0.0 ? radius : (frame ? -frame[3] : dec_double(sc->enc_dmax));
    sc->torus_side = torus_side;
    if (torus_side > 0.0) {
        // toroidal lattice of [0, side)^3 (R52, as R19): D = floor(side / R) >= 3 boxes of
        // edge L = side / D per axis, origin 0; boxes are clamped to D - 1 in k_key (R20)
        const double Dd = floor(torus_side / R);
        const bool bad = !(R > 0.0) || !(Dd >= 3.0) || !(Dd < 1.0e6);
        const int D = bad ? 3 : (int)Dd;
        sc->R = R;
        sc->R2 = R * R;
        sc->L = torus_side / (double)D;
        long long ns = 64;
        for (int a = 0; a < 3; ++a) {
            sc->o[a] = 0.0;
            sc->hi[a] = torus_side;
            sc->boff[a] = 0;
            sc->dims[a] = D;
            sc->T[a] = (D + 3) >> 2;
            if (sc->tile_order) sc->T[a] = (sc->T[a] + 7) & ~7;
            ns *= (long long)sc->T[a];
        }
        sc->nslots = ns;
        if (bad) sc->overflow = 6;  // not a valid torus for this R: nothing is computed
        else if (ns >= 0xFFFFFFFFll || ns > sc->slot_cap) sc->overflow = 1;
        sc->has_frame = 0;
        sc->dmax_prev = dec_double(sc->enc_dmax);
        if (reset_after) {
            for (int a = 0; a < 3; ++a) {
                sc->enc_lo[a] = enc_double(INFINITY);
                sc->enc_hi[a] = enc_double(-INFINITY);
            }
            sc->enc_dmax = enc_double(-INFINITY);
        }
        return;
    }
    const double L = R * (1.0 + 0x1p-20);
    sc->R = R;
    sc->R2 = R * R;
    sc->L = L;
    long long ns = 64;
    bool bad = !(L > 0.0) || !isfinite(L);
    for (int a = 0; a < 3; ++a) {
        const double lo = dec_double(sc->enc_lo[a]), hi = dec_double(sc->enc_hi[a]);
        const double o = frame ? frame[a] : lo;
        sc->o[a] = o;
        sc->hi[a] = hi;
        const double b0 = frame ? floor((lo - o) / L) : 0.0;
        const double ext = floor((hi - o) / L) - b0;
        if (!(ext < 1.0e9) || !(b0 >= 0.0 && b0 < 2.0e9)) bad = true;
        sc->boff[a] = bad ? 0 : (int)b0;
        const int dim = bad ? 1 : (int)ext + 1;
        sc->dims[a] = dim;
        sc->T[a] = (dim + 3) >> 2;
        if (sc->tile_order) sc->T[a] = (sc->T[a] + 7) & ~7;  // whole 8^3 super-tiles
        ns *= (long long)sc->T[a];
        if (ns > (1ll << 40)) bad = true;
    }
    sc->nslots = ns;
    if (bad || ns >= 0xFFFFFFFFll || ns > sc->slot_cap) sc->overflow = 1;
    sc->has_frame = frame ? 1 : 0;
    sc->dmax_prev = dec_double(sc->enc_dmax);
    if (reset_after) {  // the mechanics epilogue accumulates the next step's extent
        for (int a = 0; a < 3; ++a) {
            sc->enc_lo[a] = enc_double(INFINITY);
            sc->enc_hi[a] = enc_double(-INFINITY);
        }
        sc->enc_dmax = enc_double(-INFINITY);
    }
}

bdm_status launch_grid_geometry(Ctx *c, const bdm_agents *a, const bdm_agents *g, double radius,
                                cudaStream_t st) {
    // the extent of `a` is already in the scalars when the previous mechanics step wrote
    // exactly these arrays with the fused reduction (option "fuse_reduce")
    const bool reuse = c->fuse_reduce && c->fused_valid && c->fused_x == a->x && c->fused_n == a->n;
    if (!reuse) k_reset_scalars<<<1, 32, 0, st>>>(c->sc);
    const bdm_agents *sets[2] = {reuse ? nullptr : a, g};
    for (const bdm_agents *s : sets) {
        if (!s || s->n == 0) continue;
        int64_t blocks = (s->n + 255) / 256;
        const int64_t maxb = (int64_t)c->sm_count * 8;
        if (blocks > maxb) blocks = maxb;
        k_reduce<<<(unsigned)blocks, 256, 0, st>>>(s->n, s->x, s->y, s->z, s->diameter, c->sc);
        c->launches += 1;
    }
    k_setup<<<1, 32, 0, st>>>(c->sc, radius, c->frame, c->fuse_reduce ? 1 : 0, c->torus_side);
    c->launches += reuse ? 1 : 2;
    c->fused_valid = false;
    BDM_LAUNCH_CHECK("grid geometry");
    return BDM_OK;
}

// ============================================================== a2: keys + histogram
__global__ void k_zero_counts(uint32_t *__restrict__ counts, DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->scan_epoch = sc->scan_epoch % 0x3FFFFFFFu + 1u;
    const long long m = sc->nslots + 1;
    // 16-byte stores (the array is 256-byte aligned): with 4-byte stores the kernel was
    // bound by its own instruction issue (77 %), not by the 27 MB it writes at cfg2
    const long long m4 = m >> 2;
    uint4 *const c4 = reinterpret_cast<uint4 *>(counts);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m4;
         i += (long long)gridDim.x * blockDim.x)
        c4[i] = make_uint4(0u, 0u, 0u, 0u);
    if (blockIdx.x == 0 && threadIdx.x < (m & 3)) counts[4 * m4 + threadIdx.x] = 0u;
}

// Agents [0, nl) are local, [nl, nl + ng) are the ghosts (aura) of this build.
struct Src {
    int64_t nl, ng;
    const double *__restrict__ x, *__restrict__ y, *__restrict__ z, *__restrict__ d, *__restrict__ vol;
    const uint32_t *__restrict__ id, *__restrict__ flags;
    const double *__restrict__ gx, *__restrict__ gy, *__restrict__ gz, *__restrict__ gd;
    const uint32_t *__restrict__ gid, *__restrict__ gflags;
};

// kGridIlp agents per thread (strided by the block size, so every load and store stays
// coalesced): the per-agent atomics' round trips overlap instead of one per thread
#ifndef BDM_GRID_ILP
#define BDM_GRID_ILP 4
#endif
constexpr int kGridIlp = BDM_GRID_ILP;
constexpr int kGridThreads = 256;

__global__ void __launch_bounds__(kGridThreads) k_key(Src S, const DevScalars *__restrict__ sc,
                                                      uint32_t *__restrict__ key,
                                                      uint32_t *__restrict__ rank,
                                                      uint32_t *__restrict__ counts) {
    if (sc->overflow) return;
    const int64_t n = S.nl + S.ng;
    const int64_t i0 = blockIdx.x * (int64_t)(kGridThreads * kGridIlp) + threadIdx.x;
    const double L = sc->L, o0 = sc->o[0], o1 = sc->o[1], o2 = sc->o[2];
    const int f0 = sc->boff[0], f1 = sc->boff[1], f2 = sc->boff[2], T0 = sc->T[0], T1 = sc->T[1];
    const uint16_t *const hilb = sc_hilb(sc);
    const bool torus = sc->torus_side > 0.0;
    const int Dm0 = sc->dims[0] - 1, Dm1 = sc->dims[1] - 1, Dm2 = sc->dims[2] - 1;
    uint32_t k[kGridIlp], r[kGridIlp];
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q) {
        const int64_t i = i0 + q * kGridThreads;
        k[q] = 0;
        if (i < n) {
            const bool gh = i >= S.nl;
            const int64_t j = gh ? i - S.nl : i;
            const double px = gh ? S.gx[j] : S.x[j], py = gh ? S.gy[j] : S.y[j],
                         pz = gh ? S.gz[j] : S.z[j];
            int bx = (int)floor((px - o0) / L) - f0;
            int by = (int)floor((py - o1) / L) - f1;
            int bz = (int)floor((pz - o2) / L) - f2;
            if (torus) {  // x == side (R20) and rounding at the faces: the edge boxes
                bx = bx < 0 ? 0 : (bx > Dm0 ? Dm0 : bx);
                by = by < 0 ? 0 : (by > Dm1 ? Dm1 : by);
                bz = bz < 0 ? 0 : (bz > Dm2 ? Dm2 : bz);
            }
            k[q] = box_key(bx, by, bz, T0, T1, hilb);
        }
    }
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q)
        if (i0 + q * kGridThreads < n) r[q] = atomicAdd(&counts[k[q]], 1u);
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q) {
        const int64_t i = i0 + q * kGridThreads;
        if (i < n) {
            key[i] = k[q];
            rank[i] = r[q];
        }
    }
}

// ============================================================== a3: exclusive scan
// Reduce-then-scan over m = nslots + 1 counts, tiles of 4096 (512 threads x 8).
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int l = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (l >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix and
// writes the block total to *total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t wsum[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint32_t inc = warp_incl_scan(v);
    if (l == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t s = l < nw ? wsum[l] : 0u;
        s = warp_incl_scan(s);
        wsum[l] = s;  // inclusive prefix over warps
    }
    __syncthreads();
    const uint32_t before = (w > 0 ? wsum[w - 1] : 0u) + inc - v;
    *total = wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

// m = nslots + 1 from the device scalars (grid scan) or the explicit m_host (sc == nullptr)
__device__ __forceinline__ long long scan_len(const DevScalars *__restrict__ sc, long long m_host) {
    return sc ? sc->nslots + 1 : m_host;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *__restrict__ cnt,
                                                              uint32_t *__restrict__ bsum,
                                                              const DevScalars *__restrict__ sc,
                                                              long long m_host) {
    if (sc && sc->overflow) return;
    const long long m = scan_len(sc, m_host);
    const long long base = (long long)blockIdx.x * kScanTile;
    if (base >= m) return;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + (long long)k * kScanThreads + threadIdx.x;
        if (i < m) s += cnt[i];
    }
    uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// One block scans the block sums (exclusive, in place).
__global__ void __launch_bounds__(1024) k_scan_top(uint32_t *__restrict__ bsum,
                                                   const DevScalars *__restrict__ sc,
                                                   long long m_host) {
    if (sc && sc->overflow) return;
    const long long m = scan_len(sc, m_host);
    const long long nb = (m + kScanTile - 1) / kScanTile;
    const long long per = (nb + blockDim.x - 1) / blockDim.x;
    const long long b0 = threadIdx.x * per;
    uint32_t s = 0;
    for (long long b = b0; b < b0 + per && b < nb; ++b) s += bsum[b];
    uint32_t tot;
    uint32_t run = block_excl_scan(s, &tot);
    for (long long b = b0; b < b0 + per && b < nb; ++b) {
        const uint32_t v = bsum[b];
        bsum[b] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(uint32_t *__restrict__ cnt,
                                                             const uint32_t *__restrict__ bsum,
                                                             const DevScalars *__restrict__ sc,
                                                             long long m_host) {
    if (sc && sc->overflow) return;
    const long long m = scan_len(sc, m_host);
    const long long base = (long long)blockIdx.x * kScanTile;
    if (base >= m) return;
    // thread t owns items base + t*8 .. +7 (contiguous, 32 B: two 16-byte accesses when
    // the whole run is in range)
    static_assert(kScanItems == 8, "vector path assumes 8 items per thread");
    uint32_t v[kScanItems];
    const long long i0 = base + (long long)threadIdx.x * kScanItems;
    const bool full = i0 + kScanItems <= m;
    if (full) {
        const uint4 a = *reinterpret_cast<const uint4 *>(cnt + i0);
        const uint4 b = *reinterpret_cast<const uint4 *>(cnt + i0 + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = (i0 + k < m) ? cnt[i0 + k] : 0u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += v[k];
    uint32_t tot;
    uint32_t run = block_excl_scan(s, &tot) + bsum[blockIdx.x];
    uint32_t o[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        o[k] = run;
        run += v[k];
    }
    if (full) {
        *reinterpret_cast<uint4 *>(cnt + i0) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4 *>(cnt + i0 + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (i0 + k < m) cnt[i0 + k] = o[k];
    }
}

// Single-pass exclusive scan of the slot counts (decoupled look-back): tile b (kS1Tile
// counts, blockIdx order) publishes its aggregate, then its inclusive prefix once the
// prefixes before it are known; warp 0 looks back over the predecessors 32 at a time.
// One word per tile: epoch << 34 | status << 32 | value (status 1 = aggregate, 2 =
// inclusive prefix; a word of another epoch is "not ready"), so the array is never
// cleared (the epoch is bumped on the device by k_zero_counts, so a replayed CUDA
// graph tags every scan afresh).  Counts sum to the agent count (< 2^32).  Relies on tiles being dispatched in
// blockIdx order, so a tile only waits for tiles that are resident or done.
constexpr unsigned long long kScanAgg = 1ull, kScanInc = 2ull;
// Its tiles hold kS1Items counts per thread: the look-back is a serial chain of one L2
// round trip per 32 tiles, so the time falls with the tile count (8,192-count tiles:
// 812 tiles at cfg2 instead of 1,623; ncu 34.3 -> see profiles/r02/s4/ab_session4.txt).
#ifndef BDM_S1_ITEMS
#define BDM_S1_ITEMS 16
#endif
constexpr int kS1Items = BDM_S1_ITEMS;
constexpr int kS1Tile = kScanThreads * kS1Items;
static_assert(kS1Items % 4 == 0, "vector path moves 4 counts at a time");
__device__ __forceinline__ unsigned long long scan_word(uint32_t epoch, unsigned long long st,
                                                        uint32_t v) {
    return ((unsigned long long)epoch << 34) | (st << 32) | v;
}
__global__ void __launch_bounds__(kScanThreads) k_scan_single(uint32_t *__restrict__ cnt,
                                                              unsigned long long *state,
                                                              const DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    const uint32_t epoch = sc->scan_epoch;  // 1 .. 2^30 - 1 (0 = never written)
    const long long m = sc->nslots + 1;
    const long long base = (long long)blockIdx.x * kS1Tile;
    if (base >= m) return;
    uint32_t v[kS1Items];
    const long long i0 = base + (long long)threadIdx.x * kS1Items;
    const bool full = i0 + kS1Items <= m;
    if (full) {
#pragma unroll
        for (int q = 0; q < kS1Items / 4; ++q) {
            const uint4 a = *reinterpret_cast<const uint4 *>(cnt + i0 + 4 * q);
            v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kS1Items; ++k) v[k] = (i0 + k < m) ? cnt[i0 + k] : 0u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kS1Items; ++k) s += v[k];
    uint32_t tot;
    const uint32_t before = block_excl_scan(s, &tot);
    __shared__ uint32_t tile_prefix;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        volatile unsigned long long *vs = state;
        const long long b = blockIdx.x;
        if (b == 0) {
            if (lane == 0) {
                vs[0] = scan_word(epoch, kScanInc, tot);
                tile_prefix = 0u;
            }
        } else {
            if (lane == 0) vs[b] = scan_word(epoch, kScanAgg, tot);
            uint32_t excl = 0;
            long long j = b - 1;  // lane l looks at tile j - l
            for (;;) {
                const long long t = j - lane;
                unsigned long long w = t >= 0 ? vs[t] : scan_word(epoch, kScanInc, 0u);
                uint32_t st = (uint32_t)(w >> 34) == epoch ? (uint32_t)((w >> 32) & 3u) : 0u;
                while (__any_sync(0xffffffffu, st == 0u)) {  // wait for every predecessor's word
                    if (st == 0u) {
                        w = vs[t];
                        st = (uint32_t)(w >> 34) == epoch ? (uint32_t)((w >> 32) & 3u) : 0u;
                    }
                }
                const unsigned inc = __ballot_sync(0xffffffffu, st == (uint32_t)kScanInc);
                // the nearest inclusive prefix ends the look-back: sum lanes 0..k
                const int k = inc ? __ffs(inc) - 1 : 31;
                uint32_t val = lane <= k ? (uint32_t)w : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                excl += val;
                if (inc) break;
                j -= 32;
            }
            if (lane == 0) {
                __threadfence();
                vs[b] = scan_word(epoch, kScanInc, excl + tot);
                tile_prefix = excl;
            }
        }
    }
    __syncthreads();
    uint32_t run = tile_prefix + before;
    uint32_t o[kS1Items];
#pragma unroll
    for (int k = 0; k < kS1Items; ++k) {
        o[k] = run;
        run += v[k];
    }
    if (full) {
#pragma unroll
        for (int q = 0; q < kS1Items / 4; ++q)
            *reinterpret_cast<uint4 *>(cnt + i0 + 4 * q) = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kS1Items; ++k)
            if (i0 + k < m) cnt[i0 + k] = o[k];
    }
}

// ============================================================== a4: scatter + order + gather
__global__ void __launch_bounds__(kGridThreads) k_scatter(Src S, const uint32_t *__restrict__ key,
                                                          const uint32_t *__restrict__ rank,
                                                          const uint32_t *__restrict__ box_start,
                                                          uint32_t *__restrict__ perm_tmp,
                                                          uint32_t *__restrict__ skey,
                                                          uint32_t *__restrict__ sid,
                                                          const DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    const int64_t n = S.nl + S.ng;
    const int64_t i0 = blockIdx.x * (int64_t)(kGridThreads * kGridIlp) + threadIdx.x;
    uint32_t k[kGridIlp], slot[kGridIlp], id[kGridIlp];
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q) {
        const int64_t i = i0 + q * kGridThreads;
        if (i < n) {
            k[q] = key[i];
            slot[q] = rank[i];
            id[q] = i >= S.nl ? S.gid[i - S.nl] : S.id[i];
        }
    }
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q)
        if (i0 + q * kGridThreads < n) slot[q] += box_start[k[q]];
#pragma unroll
    for (int q = 0; q < kGridIlp; ++q) {
        const int64_t i = i0 + q * kGridThreads;
        if (i < n) {
            perm_tmp[slot[q]] = (uint32_t)i;
            skey[slot[q]] = k[q];
            sid[slot[q]] = id[q];
        }
    }
}

// Slot s of the scatter holds an agent of box k in arbitrary order; its final slot
// is box_start[k] + #(agents of box k with a smaller id).  Gathers the SoA there.
// Ghosts are marked with kGhost in the sorted flags; with ghosts, lflag[dst] = 1 for
// local agents (scanned afterwards into their output index).
// kFixIlp slots per thread (strided by the block size): their dependent chains (key ->
// box range -> id rank -> source -> SoA) overlap.
#ifndef BDM_FIX_ILP
#define BDM_FIX_ILP 2
#endif
constexpr int kFixIlp = BDM_FIX_ILP;
__global__ void __launch_bounds__(kGridThreads) k_fix_gather(
    Src S, const uint32_t *__restrict__ skey, const uint32_t *__restrict__ sid,
    const uint32_t *__restrict__ perm_tmp, const uint32_t *__restrict__ box_start,
    double *__restrict__ sx, double *__restrict__ sy, double *__restrict__ sz,
    double *__restrict__ sd, uint32_t *__restrict__ sidf, uint32_t *__restrict__ sflags,
    double *__restrict__ svol, uint32_t *__restrict__ lflag, uint32_t *__restrict__ perm,
    const DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    const int64_t n = S.nl + S.ng;
    const int64_t s0 = blockIdx.x * (int64_t)(kGridThreads * kFixIlp) + threadIdx.x;
    uint32_t lo[kFixIlp], hi[kFixIlp], me[kFixIlp], src[kFixIlp];
#pragma unroll
    for (int q = 0; q < kFixIlp; ++q) {
        const int64_t s = s0 + q * kGridThreads;
        if (s == n && lflag) lflag[n] = 0u;
        if (s < n) {
            const uint32_t k = skey[s];
            lo[q] = box_start[k];
            hi[q] = box_start[k + 1];
            me[q] = sid[s];
            src[q] = perm_tmp[s];
        }
    }
#pragma unroll
    for (int q = 0; q < kFixIlp; ++q) {
        const int64_t s = s0 + q * kGridThreads;
        if (s >= n) continue;
        uint32_t r = 0;
        for (uint32_t t = lo[q]; t < hi[q]; ++t) r += (sid[t] < me[q]);
        lo[q] += r;  // the destination slot
    }
#pragma unroll
    for (int q = 0; q < kFixIlp; ++q) {
        const int64_t s = s0 + q * kGridThreads;
        if (s >= n) continue;
        const uint32_t dst = lo[q], sr = src[q];
        if (perm) perm[dst] = sr;  // sort_every != 1: the mechanics writes back to src
        if ((int64_t)sr < S.nl) {
            sx[dst] = S.x[sr];
            sy[dst] = S.y[sr];
            sz[dst] = S.z[sr];
            sd[dst] = S.d[sr];
            sflags[dst] = S.flags[sr];
            if (S.vol) svol[dst] = S.vol[sr];
            if (lflag) lflag[dst] = 1u;
        } else {
            const int64_t j = (int64_t)sr - S.nl;
            sx[dst] = S.gx[j];
            sy[dst] = S.gy[j];
            sz[dst] = S.gz[j];
            sd[dst] = S.gd[j];
            sflags[dst] = S.gflags[j] | kGhost;
            if (S.vol) svol[dst] = 0.0;
            lflag[dst] = 0u;
        }
        sidf[dst] = me[q];
    }
}

bdm_status launch_grid_sort(Ctx *c, const bdm_agents *a, const bdm_agents *g, cudaStream_t st) {
    Src S;
    S.nl = a->n;
    S.ng = g ? g->n : 0;
    S.x = a->x; S.y = a->y; S.z = a->z; S.d = a->diameter; S.vol = a->volume;
    S.id = a->id; S.flags = a->flags;
    S.gx = g ? g->x : nullptr; S.gy = g ? g->y : nullptr; S.gz = g ? g->z : nullptr;
    S.gd = g ? g->diameter : nullptr; S.gid = g ? g->id : nullptr;
    S.gflags = g ? g->flags : nullptr;
    const int64_t n = S.nl + S.ng;
    {
#ifndef BDM_ZERO_BLOCKS_PER_SM
#define BDM_ZERO_BLOCKS_PER_SM 4
#endif
        int64_t zb = ((c->slot_cap + 1) / 4 + 1 + 1023) / 1024;  // one 16-byte store per thread and pass
        const int64_t maxb = (int64_t)c->sm_count * BDM_ZERO_BLOCKS_PER_SM;
        if (zb > maxb) zb = maxb;
        k_zero_counts<<<(unsigned)zb, 1024, 0, st>>>(c->box_start, c->sc);
    }
    bdm_status s;
    if (S.vol && (s = need_agent_buf(c, &c->svol)) != BDM_OK) return s;
    if (S.ng > 0 && (s = need_agent_buf(c, &c->lrank)) != BDM_OK) return s;
    // row f1: physically reorder the caller's SoA only on every sort_every-th build
    // (0: never); otherwise the mechanics writes each agent back to its input index
    c->keep_order = c->sort_every != 1 &&
                    (c->sort_every == 0 || c->grid_builds % c->sort_every != 0);
    ++c->grid_builds;
    if (c->keep_order && (s = need_agent_buf(c, &c->perm)) != BDM_OK) return s;
    const unsigned nbi = (unsigned)((n + kGridThreads * kGridIlp - 1) / (kGridThreads * kGridIlp));
    k_key<<<nbi, kGridThreads, 0, st>>>(S, c->sc, c->key, c->rank, c->box_start);
    const unsigned sb = (unsigned)((c->slot_cap + 1 + kS1Tile - 1) / kS1Tile);
    if (c->scan_state_cap < (int64_t)sb) {
        if (c->scan_state) cudaFree(c->scan_state);
        c->scan_state = nullptr;
        c->scan_state_cap = 0;
        BDM_CUDA_TRY(cudaMalloc(&c->scan_state, (size_t)sb * sizeof(unsigned long long)));
        BDM_CUDA_TRY(cudaMemsetAsync(c->scan_state, 0, (size_t)sb * sizeof(unsigned long long), st));
        c->scan_state_cap = sb;
    }
    k_scan_single<<<sb, kScanThreads, 0, st>>>(c->box_start, c->scan_state, c->sc);
    k_scatter<<<nbi, kGridThreads, 0, st>>>(S, c->key, c->rank, c->box_start, c->perm_tmp, c->skey,
                                            c->sid, c->sc);
    uint32_t *lflag = S.ng > 0 ? c->lrank : nullptr;
    k_fix_gather<<<(unsigned)((n + 1 + kGridThreads * kFixIlp - 1) / (kGridThreads * kFixIlp)),
                   kGridThreads, 0, st>>>(
        S, c->skey, c->sid, c->perm_tmp, c->box_start, c->sx, c->sy, c->sz, c->sd, c->sidf,
        c->sflags, c->svol, lflag, c->keep_order ? c->perm : nullptr, c->sc);
    c->launches += 5;
    BDM_LAUNCH_CHECK("grid sort");
    if (S.ng > 0) return launch_scan_u32(c, c->lrank, n + 1, st);  // output index of locals
    return BDM_OK;
}

int64_t scan_block_count(int64_t slot_cap) { return (slot_cap + 1 + kScanTile - 1) / kScanTile; }

// Exclusive scan of m values in place (block sums in the context's scan buffer, which
// bdm_reserve / grow_agents size for max(slots, agents) + 1 entries).
bdm_status launch_scan_u32(Ctx *c, uint32_t *data, long long m, cudaStream_t st) {
    if (m <= 0) return BDM_OK;
    const unsigned sb = (unsigned)((m + kScanTile - 1) / kScanTile);
    if ((int64_t)sb + 1 > c->block_sums_cap) {
        set_error("scan buffer too small");
        return BDM_ECAPACITY;
    }
    k_scan_reduce<<<sb, kScanThreads, 0, st>>>(data, c->block_sums, nullptr, m);
    k_scan_top<<<1, 1024, 0, st>>>(c->block_sums, nullptr, m);
    k_scan_apply<<<sb, kScanThreads, 0, st>>>(data, c->block_sums, nullptr, m);
    c->launches += 3;
    BDM_LAUNCH_CHECK("scan");
    return BDM_OK;
}

}  // namespace bdm
