// kernels_row.cu -- the mechanics step as a row-broadcast tile kernel.
//
//   a5  static classification: pull test over the neighbours' last-step
//       flags, only for agents whose own flags allow it; static agents skip the force
//   a6  27-box candidate scan, radius filter D <= R^2
//   a7  Eq. 4.1/4.2 pair force, summed in the canonical order (R9)
//   a8  displacement dt*F, threshold, cap; write-back + flags
//   a9  boundary: open / closed
//
// Work unit: a tile of 2 x 4 x 8 boxes (x, y, z).  The tile and its one-box halo (a
// 4 x 6 x 10-box region) are staged in shared memory in row-major box order (z, y, x),
// ids ascending inside a box, so for every agent "canonical order" (R9: boxes in
// (dz, dy, dx) order, ascending id in a box) is "ascending staged index".
//
// The tile's 32 x-rows (2 boxes each) are the broadcast units.  The candidates of a
// row are the agents of the 9 region rows (y-1..y+1, z-1..z+1), which are three
// contiguous staged ranges (one per z: the three region rows of one z are adjacent).
// A warp loads the row's candidates into registers (lane l holds positions l, l+32,
// l+64, l+96; pairs packed for the f32x2 pipe), then for each own agent of the row,
// with the agent's coordinates broadcast, tests all candidate positions at once and
// takes the survivors as ballot words: the words, concatenated, are the agent's
// survivor set in canonical order.  The test is a conservative fp32 contact test
//       D32 <= min((r'_i + r'_j)^2, R2f),  r' = fl32(r + 2^-16 L),  R2f = R^2 (1 + 2^-12)
// on region-relative coordinates (never rejects a true contact; see below), or the
// neighbour test D32 <= R2f for agents that need their whole neighbour set (static
// candidates, counters).  Rows' agents are gathered into groups of <= 32 (one lane per
// agent); per group:
//   expand  lane k lists its survivors (staged index | k << 9) in canonical order
//   pull    (static candidates only) exact D <= R^2 and the neighbours' changed flags
//   force   lane-parallel over the group's survivors, 64 at a time: the exact fp64 D,
//           the neighbour and contact tests and Eq. 4.1/4.2, s = F_N / dist (0 for
//           non-contacts, static owners)
//   accumulate  lane k adds its own survivors in order: F = fma(s, x_i - x_j, F); a
//           non-contact has s = 0 and fma(0, d, F) == F exactly (F never is -0)
//   finish  a8/a9 and the write-back (finish_agent)
//
// Conservative prefilter (fp32, relative to the region corner X0): |x - X0| <= 10.01 L,
// so each staged coordinate carries <= 2^-24 16 L = 2^-20 L of rounding and a
// difference <= 2^-19 L; with the fp32 rounding of the squares, D32 <= (rho +
// sqrt(3) 2^-19 L)^2 (1 + 2^-22) for real distance rho.  A counted contact has
// rho < (r_i + r_j)(1 + 2^-49) and rho <= R(1 + 2^-50); the threshold is >= (r_i + r_j +
// 2^-15 L)^2 (1 - 2^-21.4) >= that bound whenever r_i + r_j <= L (and when r_i + r_j >
// L >= R it exceeds the bound through rho <= R), with a margin of about 8x.  The
// neighbour threshold R2f has the same 36x margin over D32 <= R^2 (1 + 6.6e-6).
// Preconditions checked per launch: |coordinates| / L < 2^30, 2^-60 < L < 2^60; else
// every tile takes the reference formulation.
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"
#include "mech_common.cuh"

namespace bdm {

constexpr int kRW = 2, kRY = 4, kRZ = 8;                        // tile, boxes
constexpr int kRGX = kRW + 2, kRGY = kRY + 2, kRGZ = kRZ + 2;   // region 4 x 6 x 10
constexpr int kRNB = kRGX * kRGY * kRGZ;                        // 240 region boxes
constexpr int kRSQ = (kRNB + 31) / 32;                          // scan items per lane
constexpr int kRThreads = 128, kRWarps = kRThreads / 32;
constexpr int kRMax = 480;      // staged agents per region (mean 382, sd 20 at cfg2)
constexpr int kRP = 4;          // candidate words per row (128 positions)
constexpr int kRECap = 256;     // survivors per group
constexpr int kRCh = 64;        // survivors per force chunk
constexpr float kRSent = 1e30f;

struct RowWarp {
    uint16_t ea[kRECap];        // survivor: staged index m | group agent k << 9
    double es[kRCh];            // s = F_N / dist of the chunk's survivors (0: none)
    uint8_t ef[kRCh];           // bit0 F_N != 0, bit1 contact, bit2 neighbour
    uint4 mask[32];             // ballot words per group agent (words >= P are 0)
    float4 dup[32];             // the row's own agents: x, y, z, r' (or sentinels)
    uint16_t ga[32];            // group agent -> staged index
    uint16_t sg[32][5];         // position -> staged index: s0, b1, d1, b2, d2
    uint32_t gf[32];            // group agent flags (start of step)
    uint8_t chg[32];            // static candidate saw a changed neighbour
    double ext[7];
    unsigned long long cnt[5];
};

struct RowSmem {
    GridView g;
    float R2f;
    int use_pf, edge_only, dbg;
    int next_tile[2];
    int row_next;                   // dynamic row assignment within the tile
    int lo_box[3], hi_box[3];
    uint32_t start[kRNB];
    uint32_t off[kRNB + 4];
    uint8_t mbox[kRMax];        // staged index -> region box
    float4 P[kRMax + 1];        // fp32 region-relative x, y, z and r'; sentinel at M
    double X[kRMax], Y[kRMax], Z[kRMax], Rr[kRMax];
    RowWarp W[kRWarps];
};

__device__ __forceinline__ unsigned long long rpk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void rupk(unsigned long long v, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}

// Candidate pair (two positions) in packed registers.
struct CPair {
    unsigned long long x, y, z, r;
};
__device__ __forceinline__ CPair cpair(float4 p, float4 q) {
    return CPair{rpk(p.x, q.x), rpk(p.y, q.y), rpk(p.z, q.z), rpk(p.w, q.w)};
}

// Survivor bits of the agent (ax, ay, az, ar) against a candidate pair: f32x2 squared
// distances (per element the scalar fl(fma(dz,dz, fma(dy,dy, dx*dx)))) against the
// per-pair threshold.
template <bool kStats>
__device__ __forceinline__ void test_pair(unsigned long long axx, unsigned long long ayy,
                                          unsigned long long azz, unsigned long long arr,
                                          const CPair &c, float R2f, bool &p0, bool &p1) {
    unsigned long long ex, ey, ez, d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ex) : "l"(axx), "l"(c.x));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ey) : "l"(ayy), "l"(c.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ez) : "l"(azz), "l"(c.z));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(d) : "l"(ex));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(ey), "l"(d));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(ez), "l"(d));
    float d0, d1;
    rupk(d, d0, d1);
    if (kStats) {
        p0 = d0 <= R2f;
        p1 = d1 <= R2f;
    } else {
        unsigned long long s, t;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(arr), "l"(c.r));
        asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(t) : "l"(s));
        float t0, t1;
        rupk(t, t0, t1);
        p0 = d0 <= fminf(t0, R2f);
        p1 = d1 <= fminf(t1, R2f);
    }
}
// One row: fill the candidate words (lane holds positions lane + 32 u, u < NP, as f32x2
// pairs (u, u + 1)), then test every own agent of the row against all of them.  NP = 2
// or 4 words (64 or 128 positions; positions past nc hold the sentinel).
template <bool kStats, int NP>
__device__ __forceinline__ void row_tests(const RowSmem &S, RowWarp &Wp, int gn, int na,
                                          int nc, int s0, int b1, int d1, int b2, int d2,
                                          int M, float R2f, int lane) {
    float4 q[NP];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
        const int p = 32 * u + lane;
        const int m = p >= nc ? M : (p < b1 ? s0 + p : (p < b2 ? d1 + p : d2 + p));
        q[u] = S.P[m];
    }
    const CPair c01 = cpair(q[0], q[1]);
    CPair c23;
    if (NP == 4) c23 = cpair(q[2], q[3]);
#pragma unroll 2
    for (int j = 0; j < na; ++j) {
        const float4 a = Wp.dup[j];
        const unsigned long long axx = rpk(a.x, a.x), ayy = rpk(a.y, a.y), azz = rpk(a.z, a.z),
                                 arr = rpk(a.w, a.w);
        bool p0, p1;
        test_pair<kStats>(axx, ayy, azz, arr, c01, R2f, p0, p1);
        const uint32_t b0 = __ballot_sync(0xffffffffu, p0), bb1 = __ballot_sync(0xffffffffu, p1);
        uint32_t bb2 = 0, bb3 = 0;
        if (NP == 4) {
            test_pair<kStats>(axx, ayy, azz, arr, c23, R2f, p0, p1);
            bb2 = __ballot_sync(0xffffffffu, p0);
            bb3 = __ballot_sync(0xffffffffu, p1);
        }
        if (lane == (j & 31)) Wp.mask[gn + j] = make_uint4(b0, bb1, bb2, bb3);
    }
}

// Exact fp64 part of one survivor (owner staged a, candidate m): the canonical D, the
// neighbour test, the contact test and Eq. 4.1/4.2.  Returns s (0 unless a contact)
// and the flags bit0 F_N != 0, bit1 contact, bit2 neighbour.
__device__ __forceinline__ double pair_force(const RowSmem &S, const MechArgs &A, int a, int m,
                                             uint32_t &fl) {
    const double ex = S.X[a] - S.X[m], ey = S.Y[a] - S.Y[m], ez = S.Z[a] - S.Z[m];
    const double D = fma(ez, ez, fma(ey, ey, ex * ex));
    const bool nbr = D <= S.g.R2;
    const double ri = S.Rr[a], rj = S.Rr[m];
    const double dist = sqrt(D);
    const double del = (ri + rj) - dist;
    const double rb = (ri * rj) / (ri + rj);
    const double Fn = A.k * del - A.gamma * sqrt(rb * del);
    const double s = Fn / dist;
    const bool cont = nbr && del > 0.0 && dist > 0.0;
    fl = (nbr ? 4u : 0u) | (cont ? (2u | (Fn != 0.0 ? 1u : 0u)) : 0u);
    return cont ? s : 0.0;
}

// debug marker (option prefilter bit 3): the flags of an agent's output slot record the
// tile and the path that wrote it
__device__ __forceinline__ void dbg_mark(const MechArgs &A, uint32_t gi, int t, int path) {
    A.oflags[gi] = 0x80000000u | ((uint32_t)t << 8) | (uint32_t)path;
}

__device__ __forceinline__ uint32_t staged_gi(const RowSmem &S, int m) {
    const int lb = S.mbox[m];
    return S.start[lb] + (uint32_t)m - S.off[lb];
}

// The reference formulation for one agent (rare paths: crowded rows, groups with more
// survivors than the buffer, over-full regions), out of line to keep the kernel's hot
// loops small in the instruction cache.
__device__ __noinline__ void row_slow(const MechArgs &A, const GridView &g, uint32_t gi,
                                      Counts &c) {
    mech_agent_global(A, g, gi, c);
}

// Merges a group's counters into the warp's shared accumulators (lane 0 writes); out of
// line (the fp64 min/max shuffles are long), and only called when there is something to
// merge (edge tiles of the fused extent, counters).
template <bool kStats>
__device__ __noinline__ void row_merge_ool(const Counts &c, RowWarp &Wp, int sides, int lane) {
    if (sides) {
        const double v0[7] = {c.lo0, c.lo1, c.lo2, c.hi0, c.hi1, c.hi2, c.dmax};
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            if (!((sides >> q) & 1)) continue;
            double v = v0[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double t = __shfl_xor_sync(0xffffffffu, v, o);
                v = q < 3 ? fmin(v, t) : fmax(v, t);
            }
            if (lane == 0) Wp.ext[q] = q < 3 ? fmin(Wp.ext[q], v) : fmax(Wp.ext[q], v);
        }
    }
    if (kStats) {
        const unsigned long long a = warp_sum_u64(c.cand), b = warp_sum_u64(c.nbr),
                                 d = warp_sum_u64(c.cont), e = warp_sum_u64(c.stat),
                                 f = warp_sum_u64(c.moved);
        if (lane == 0) {
            Wp.cnt[0] += a;
            Wp.cnt[1] += b;
            Wp.cnt[2] += d;
            Wp.cnt[3] += e;
            Wp.cnt[4] += f;
        }
    }
    __syncwarp();
}
template <bool kStats>
__device__ __forceinline__ void row_merge(const Counts &c, RowWarp &Wp, int sides, int lane) {
    if (sides || kStats) row_merge_ool<kStats>(c, Wp, sides, lane);
}

// One group of gn <= 32 own agents (lane k = group agent k).
template <bool kStats>
__device__ __forceinline__ void row_group(const MechArgs &A, const RowSmem &S, RowWarp &Wp,
                                          int gn, int sides, int lane, int tile) {
    Counts c;
    const int k = lane;
    bool act = false, cs = false;
    int a = 0;
    uint32_t fi = 0, m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    if (k < gn) {
        fi = Wp.gf[k];
        act = !(fi & kGhost);
        a = Wp.ga[k];
        if (act) {
            cs = A.detect_static && !(fi & kChanged) && ((fi >> BDM_FLAG_NNZ_SHIFT) & 3u) <= 1u;
            const uint4 mk = Wp.mask[k];
            m0 = mk.x; m1 = mk.y; m2 = mk.z; m3 = mk.w;
        }
    }
    // survivors (the own position is always among them: D32 = 0)
    const int cnt = act ? __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3) - 1 : 0;
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const int lo = inc - cnt, hi = inc;
    const int E = __shfl_sync(0xffffffffu, inc, 31);
    if (E > kRECap || (S.dbg & 1)) {  // more survivors than the buffer: reference formulation
        if (act) {
            row_slow(A, S.g, staged_gi(S, a), c);
            if (S.dbg & 4) dbg_mark(A, staged_gi(S, a), tile, 3);
        }
        row_merge<kStats>(c, Wp, sides, lane);
        return;
    }
    // ---- expand: position p -> staged index, canonical order, self excluded
    {
        const uint16_t *sgk = Wp.sg[k < 32 ? k : 0];
        const int s0 = sgk[0], b1 = sgk[1], d1 = sgk[2], b2 = sgk[3], d2 = sgk[4];
        const int trip = __reduce_max_sync(0xffffffffu, cnt + (act ? 1 : 0));
        int pos = lo;
        for (int it = 0; it < trip; ++it) {
            const int wsel = m0 ? 0 : (m1 ? 1 : (m2 ? 2 : 3));
            const uint32_t bits = m0 ? m0 : (m1 ? m1 : (m2 ? m2 : m3));
            if (bits) {
                const int p = 32 * wsel + (__ffs(bits) - 1);
                const uint32_t nb = bits & (bits - 1u);
                if (wsel == 0) m0 = nb;
                else if (wsel == 1) m1 = nb;
                else if (wsel == 2) m2 = nb;
                else m3 = nb;
                const int m = p < b1 ? s0 + p : (p < b2 ? d1 + p : d2 + p);
                if (m != a) Wp.ea[pos++] = (uint16_t)(m | (k << 9));
            }
        }
    }
    if (act) Wp.chg[k] = 0;
    __syncwarp();
    // ---- a5 pull test for static candidates: exact neighbours with a changed flag
    const unsigned cs_mask = __ballot_sync(0xffffffffu, cs);
    bool is_static = false;
    if (cs_mask) {
        for (int e = lane; e < E; e += 32) {
            const uint32_t ev = Wp.ea[e];
            const int k2 = (int)(ev >> 9), m = (int)(ev & 511u);
            if (!((cs_mask >> k2) & 1u)) continue;
            const int a2 = Wp.ga[k2];
            const double ex = S.X[a2] - S.X[m], ey = S.Y[a2] - S.Y[m], ez = S.Z[a2] - S.Z[m];
            const double D = fma(ez, ez, fma(ey, ey, ex * ex));
            if (D <= S.g.R2 && (A.sflags[staged_gi(S, m)] & kChanged)) Wp.chg[k2] = 1;
        }
        __syncwarp();
        is_static = cs && !Wp.chg[k];
    }
    const unsigned stat_mask = __ballot_sync(0xffffffffu, is_static);
    // ---- force chunks, then the ordered accumulation of the own survivors
    double xi = 0.0, yi = 0.0, zi = 0.0;
    if (act) {
        xi = S.X[a];
        yi = S.Y[a];
        zi = S.Z[a];
    }
    double Fx = 0.0, Fy = 0.0, Fz = 0.0;
    int nnz = 0;
    uint32_t my_cont = 0, my_nbr = 0;
    for (int c0 = 0; c0 < E; c0 += kRCh) {  // warp-uniform
        {
            const int e1 = c0 + lane, e2 = c0 + 32 + lane;
            const bool h1 = e1 < E, h2 = e2 < E;
            const uint32_t ev1 = h1 ? Wp.ea[e1] : 0u, ev2 = h2 ? Wp.ea[e2] : 0u;
            const int k1 = (int)(ev1 >> 9), k2 = (int)(ev2 >> 9);
            const bool w1 = h1 && !((stat_mask >> k1) & 1u), w2 = h2 && !((stat_mask >> k2) & 1u);
            uint32_t f1 = 0, f2 = 0;
            double s1 = 0.0, s2 = 0.0;
            if (w1) s1 = pair_force(S, A, Wp.ga[k1], (int)(ev1 & 511u), f1);
            if (w2) s2 = pair_force(S, A, Wp.ga[k2], (int)(ev2 & 511u), f2);
            if (h1) {
                Wp.es[lane] = s1;
                Wp.ef[lane] = (uint8_t)f1;
            }
            if (h2) {
                Wp.es[32 + lane] = s2;
                Wp.ef[32 + lane] = (uint8_t)f2;
            }
        }
        __syncwarp();
        const int e_lo = lo > c0 ? lo : c0, e_hi = hi < c0 + kRCh ? hi : c0 + kRCh;
        for (int e = e_lo; e < e_hi; ++e) {
            const int m = (int)(Wp.ea[e] & 511u);
            const double s_ = Wp.es[e - c0];
            const uint32_t f = Wp.ef[e - c0];
            Fx = fma(s_, xi - S.X[m], Fx);
            Fy = fma(s_, yi - S.Y[m], Fy);
            Fz = fma(s_, zi - S.Z[m], Fz);
            nnz += (int)(f & 1u);
            my_cont += (f >> 1) & 1u;
            my_nbr += (f >> 2) & 1u;
        }
        __syncwarp();
    }
    if (act) {
        nnz = nnz < 2 ? nnz : 2;
        if (is_static) {
            nnz = (int)((fi >> BDM_FLAG_NNZ_SHIFT) & 3u);
        } else if (kStats) {
            // the 27-box candidates minus the agent itself (from the region's box table)
            const int lb = S.mbox[a];
            uint32_t ca = 0;
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy) {
                    const int r = lb + dz * kRGX * kRGY + dy * kRGX;
                    ca += S.off[r + 2] - S.off[r - 1];
                }
            c.cand += ca - 1u;
            c.nbr += my_nbr;
            c.cont += my_cont;
        }
        finish_agent(A, staged_gi(S, a), xi, yi, zi, Fx, Fy, Fz, is_static, nnz, c);
        if (S.dbg & 4) dbg_mark(A, staged_gi(S, a), tile, 2);
    }
    row_merge<kStats>(c, Wp, sides, lane);
}

template <bool kStats>
__global__ void __launch_bounds__(kRThreads, 6) k_mech_row(const __grid_constant__ MechArgs A,
                                                          DevScalars *__restrict__ sc,
                                                          int allow_prefilter) {
    if (sc->overflow) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RowSmem &S = *reinterpret_cast<RowSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) {
        const GridView g = load_grid(sc);
        S.g = g;
        S.R2f = (float)(g.R2 * (1.0 + 0x1p-12));
        const double amax = fmax(fmax(fmax(fabs(g.o0), fabs(g.o1)), fmax(fabs(g.o2), fabs(sc->hi[0]))),
                                 fmax(fabs(sc->hi[1]), fabs(sc->hi[2])));
        S.dbg = allow_prefilter >> 1;
        S.use_pf = (allow_prefilter & 1) && amax < 0x1p30 * g.L && g.L > 0x1p-60 && g.L < 0x1p60;
        // fused extent (a1 of the next step): only tiles within 2 max_disp (+1 box) of
        // the old extent can hold a new extremum (see k_mech_tile6)
        const double md = A.max_disp;
        S.edge_only = A.fuse && !sc->has_frame && md >= 0.0 && 2.0 * md < 0x1p20 * g.L;
        if (S.edge_only) {
            const double ov[3] = {g.o0, g.o1, g.o2};
            for (int q = 0; q < 3; ++q) {
                S.lo_box[q] = (int)floor(2.0 * md / g.L) + 1;
                S.hi_box[q] = (int)floor((sc->hi[q] - 2.0 * md - ov[q]) / g.L) - 1;
            }
            if (blockIdx.x == 0) atomicMax(&sc->enc_dmax, enc_double(sc->dmax_prev));
        }
    }
    if (lane < 7) S.W[w].ext[lane] = lane < 3 ? INFINITY : -INFINITY;
    if (lane < 5) S.W[w].cnt[lane] = 0ull;
    __syncthreads();
    const GridView &g = S.g;
    const int TX = (g.D0 + kRW - 1) / kRW, TY = (g.D1 + kRY - 1) / kRY, TZ = (g.D2 + kRZ - 1) / kRZ;
    const int ntiles = TX * TY * TZ;
    const uint16_t *const hilb = g.hilb;
    RowWarp &Wp = S.W[w];
    for (int it = 0;; ++it) {
        if (tid == 0) S.next_tile[it & 1] = (int)atomicAdd(&sc->tile_next, 1u);
        __syncthreads();
        const int t = S.next_tile[it & 1];
        if (t >= ntiles) break;
        const int tx = t % TX, ty = (t / TX) % TY, tz = t / (TX * TY);
        const int bx0 = kRW * tx - 1, by0 = kRY * ty - 1, bz0 = kRZ * tz - 1;
        // ---- box table of the region (out-of-grid boxes are empty)
        for (int lb = tid; lb < kRNB; lb += kRThreads) {
            const int gx = bx0 + lb % kRGX, gy = by0 + (lb / kRGX) % kRGY, gz = bz0 + lb / (kRGX * kRGY);
            uint32_t st = 0, cn = 0;
            if (gx >= 0 && gy >= 0 && gz >= 0 && gx < g.D0 && gy < g.D1 && gz < g.D2) {
                const uint32_t key = box_key(gx, gy, gz, g.T0, g.T1, hilb);
                st = A.box_start[key];
                cn = A.box_start[key + 1] - st;
            }
            S.start[lb] = st;
            S.off[lb] = cn;
        }
        __syncthreads();
        if (w == 0) {  // exclusive scan of the region's box counts
            uint32_t v[kRSQ], sum = 0;
#pragma unroll
            for (int q = 0; q < kRSQ; ++q) {
                const int lb = lane * kRSQ + q;
                v[q] = lb < kRNB ? S.off[lb] : 0u;
                sum += v[q];
            }
            uint32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t run = inc - sum;
#pragma unroll
            for (int q = 0; q < kRSQ; ++q) {
                const int lb = lane * kRSQ + q;
                if (lb <= kRNB) S.off[lb] = run;
                run += v[q];
            }
        }
        __syncthreads();
        const int M = (int)S.off[kRNB];
        if (M == 0) continue;  // uniform
        if (M > kRMax && S.use_pf && A.dense_list) {
            // crowded region: its boxes go to the dense-box kernel as half tiles (the
            // x-half tx & 1 of the 4x4x4-box tiles (tx/2, ty, 2tz) and (tx/2, ty, 2tz+1))
            if (S.dbg & 4)
                for (int lb = tid; lb < kRNB; lb += kRThreads) {
                    const int lx = lb % kRGX, ly = (lb / kRGX) % kRGY, lz = lb / (kRGX * kRGY);
                    if (lx >= 1 && lx <= kRW && ly >= 1 && ly <= kRY && lz >= 1 && lz <= kRZ)
                        for (uint32_t u = 0; u < S.off[lb + 1] - S.off[lb]; ++u) dbg_mark(A, S.start[lb] + u, t, 5);
                }
            if (tid == 0) {
                const int Tz0 = 2 * tz, nz = Tz0 + 1 < g.T2 ? 2 : 1;
                const unsigned q = atomicAdd(&sc->n_dense, (unsigned)nz);
                for (int u = 0; u < nz; ++u)
                    A.dense_list[q + u] = (tile_rank(tx >> 1, ty, Tz0 + u, g.T0, g.T1, hilb) << 1) |
                                          (uint32_t)(tx & 1);
            }
            __syncthreads();
            continue;
        }
        int sides = 0;
        if (S.edge_only) {
            const int blo[3] = {kRW * tx, kRY * ty, kRZ * tz};
            const int bhi[3] = {kRW * tx + kRW - 1, kRY * ty + kRY - 1, kRZ * tz + kRZ - 1};
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                sides |= (blo[q] <= S.lo_box[q]) ? (1 << q) : 0;
                sides |= (bhi[q] >= S.hi_box[q]) ? (8 << q) : 0;
            }
        } else if (A.fuse) {
            sides = 0x7F;
        }
        if (M > kRMax || !S.use_pf) {
            // over-full region or |coordinates| / L >= 2^30: reference formulation, own
            // rows of warp w (boxes x = 1, 2 of region row (1 + w, 1 + i))
            for (int i = 0; i < kRZ; ++i) {
                const int lb1 = ((1 + i) * kRGY + 1 + w) * kRGX + 1;
                const int n1 = (int)(S.off[lb1 + 1] - S.off[lb1]), n2 = (int)(S.off[lb1 + 2] - S.off[lb1 + 1]);
                for (int j0 = 0; j0 < n1 + n2; j0 += 32) {
                    Counts c;
                    const int j = j0 + lane;
                    if (j < n1 + n2) {
                        const uint32_t gi = j < n1 ? S.start[lb1] + j : S.start[lb1 + 1] + (j - n1);
                        row_slow(A, g, gi, c);
                        if (S.dbg & 4) dbg_mark(A, gi, t, 4);
                    }
                    row_merge<kStats>(c, Wp, A.fuse ? 0x7F : 0, lane);
                }
            }
            __syncthreads();
            continue;
        }
        // ---- staged index -> region box
        if (tid == 0) S.row_next = 0;
        for (int lb = tid; lb < kRNB; lb += kRThreads) {
            const uint32_t o = S.off[lb], n = S.off[lb + 1] - o;
            for (uint32_t u = 0; u < n; ++u) S.mbox[o + u] = (uint8_t)lb;
        }
        __syncthreads();
        // ---- stage the region: fp64 x, y, z, r and the fp32 prefilter copy
        {
            const double L = g.L;
            const double X0 = g.o0 + (double)(bx0 + g.b0) * L, Y0 = g.o1 + (double)(by0 + g.b1) * L,
                         Z0 = g.o2 + (double)(bz0 + g.b2) * L;
            const double hpad = 0x1p-16 * L;
            for (int m = tid; m < M; m += kRThreads) {
                const uint32_t gi = staged_gi(S, m);
                const double x = A.sx[gi], y = A.sy[gi], z = A.sz[gi], r = A.sd[gi] * 0.5;
                S.X[m] = x;
                S.Y[m] = y;
                S.Z[m] = z;
                S.Rr[m] = r;
                S.P[m] = make_float4((float)(x - X0), (float)(y - Y0), (float)(z - Z0), (float)(r + hpad));
            }
            if (tid == 0) S.P[M] = make_float4(kRSent, kRSent, kRSent, 0.f);
        }
        __syncthreads();
        // ---- rows (region row (y, z), own boxes x = 1, 2), taken by the warps in turn
        const float R2f = S.R2f;
        int gn = 0;
        for (;;) {  // rows taken dynamically (their costs vary with the agent counts)
            int r = 0;
            if (lane == 0) r = atomicAdd(&S.row_next, 1);
            r = __shfl_sync(0xffffffffu, r, 0);
            if (r >= kRY * kRZ) break;
            const int ly = 1 + r % kRY, lz = 1 + r / kRY;
            const int lbo = (lz * kRGY + ly) * kRGX;
            const int a0 = (int)S.off[lbo + 1], na = (int)S.off[lbo + 3] - a0;
            if (na == 0) continue;
            int sgs[3], sgn[3];
#pragma unroll
            for (int dz = 0; dz < 3; ++dz) {
                const int b = ((lz - 1 + dz) * kRGY + ly - 1) * kRGX;
                sgs[dz] = (int)S.off[b];
                sgn[dz] = (int)S.off[b + 3 * kRGX] - sgs[dz];
            }
            const int nc = sgn[0] + sgn[1] + sgn[2];
            if (na > 32 || nc > 32 * kRP || (S.dbg & 2)) {
                // a crowded row: reference formulation for its agents
                for (int j0 = 0; j0 < na; j0 += 32) {
                    Counts c;
                    if (j0 + lane < na) {
                        const uint32_t gi = staged_gi(S, a0 + j0 + lane);
                        row_slow(A, g, gi, c);
                        if (S.dbg & 4) dbg_mark(A, gi, t, 1);
                    }
                    row_merge<kStats>(c, Wp, sides, lane);
                }
                continue;
            }
            if (gn + na > 32) {
                __syncwarp();
                row_group<kStats>(A, S, Wp, gn, sides, lane, t);
                gn = 0;
            }
            const int b1 = sgn[0], d1 = sgs[1] - sgn[0], b2 = sgn[0] + sgn[1], d2 = sgs[2] - b2;
            if (lane < na) {
                const int a = a0 + lane;
                float4 q = S.P[a];
                const uint32_t fi = A.sflags[staged_gi(S, a)];
                const bool cs = A.detect_static && !(fi & kChanged) &&
                                ((fi >> BDM_FLAG_NNZ_SHIFT) & 3u) <= 1u;
                if (fi & kGhost) q.x = -kRSent;       // a ghost tests nothing
                else if (cs) q.w = INFINITY;          // static candidate: whole neighbour set
                Wp.dup[lane] = q;
                Wp.ga[gn + lane] = (uint16_t)a;
                Wp.gf[gn + lane] = fi;
                uint16_t *sgk = Wp.sg[gn + lane];
                sgk[0] = (uint16_t)sgs[0];
                sgk[1] = (uint16_t)b1;
                sgk[2] = (uint16_t)d1;
                sgk[3] = (uint16_t)b2;
                sgk[4] = (uint16_t)d2;
            }
            __syncwarp();
            if (nc <= 64)
                row_tests<kStats, 2>(S, Wp, gn, na, nc, sgs[0], b1, d1, b2, d2, M, R2f, lane);
            else
                row_tests<kStats, 4>(S, Wp, gn, na, nc, sgs[0], b1, d1, b2, d2, M, R2f, lane);
            gn += na;
            __syncwarp();
        }
        if (gn > 0) row_group<kStats>(A, S, Wp, gn, sides, lane, t);
        __syncthreads();  // before the next tile overwrites the staged region
    }
    if (A.fuse && lane == 0) {
        for (int q = 0; q < 3; ++q) atomicMin(&sc->enc_lo[q], enc_double(Wp.ext[q]));
        for (int q = 0; q < 3; ++q) atomicMax(&sc->enc_hi[q], enc_double(Wp.ext[3 + q]));
        atomicMax(&sc->enc_dmax, enc_double(Wp.ext[6]));
    }
    if (kStats && lane < 5) atomicAdd(&sc->stats[lane], Wp.cnt[lane]);
}

template <bool kStats>
static int row_per_sm(Ctx *c) {
    static int per_sm_dev[kMaxDevices] = {};
    int &per_sm = per_sm_dev[c->device];
    if (!per_sm) {
        const int smem = (int)sizeof(RowSmem);
        int v = 0;
        if (cudaFuncSetAttribute(k_mech_row<kStats>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_mech_row<kStats>, kRThreads, smem) !=
                cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        per_sm = v < 1 ? 1 : v;
    }
    return per_sm;
}

bdm_status launch_mech_row(Ctx *c, const MechArgs &A, bool stats, cudaStream_t st) {
    const int per_sm = stats ? row_per_sm<true>(c) : row_per_sm<false>(c);
    if (!per_sm) {
        set_error("row kernel setup failed");
        return BDM_ECUDA;
    }
    const int smem = (int)sizeof(RowSmem);
    const unsigned grid = (unsigned)(c->sm_count * per_sm);
    if (stats) k_mech_row<true><<<grid, kRThreads, smem, st>>>(A, c->sc, c->prefilter);
    else k_mech_row<false><<<grid, kRThreads, smem, st>>>(A, c->sc, c->prefilter);
    return BDM_OK;
}

}  // namespace bdm
