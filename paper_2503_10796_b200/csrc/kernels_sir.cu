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
//                  S/I/R counts.  A warp handles two 32-agent slices per iteration
//                  (loads first); infection queries are compacted into a per-warp queue,
//                  32 at a time take the coarse test one per lane, and each that passes
//                  is searched by the whole warp (one of the 27 boxes per lane)
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

constexpr int kCoarse = 16;                  // fine boxes per coarse block (per axis)
constexpr uint32_t kNone = 0xFFFFFFFFu;
// Hash slots carry the step stamp in their upper 24 bits, so the table never needs
// clearing: a slot whose stamp is not the current one is empty.  Box keys need
// <= 39 bits (D <= 8192).
constexpr int kStampShift = 40;

struct SirArgs {
    int64_t n;
    double *__restrict__ x;
    double *__restrict__ y;
    double *__restrict__ z;
    uint8_t *__restrict__ state;
    const uint32_t *__restrict__ id;  // nullable: id = index
    double side, L, R2, half, p_inf, p_rec;
    unsigned long long t_inf, t_rec;  // uniform32(w) < p  <=>  w < t = ceil(p 2^32) (host)
    double Rq, invC;                  // coarse test: padded radius, 1 / (16 L)
    int D, B, cf;                     // fine boxes / coarse blocks per axis; boxes per block
    uint32_t k0, k1, step;
    uint32_t rk0[10], rk1[10];        // Philox round keys k + r (0x9E3779B9, 0xBB67AE85)
    // infected index
    unsigned long long *__restrict__ keys;   // stamp << 40 | box key
    unsigned long long *__restrict__ heads;  // stamp << 32 | first infected slot
    unsigned long long stamp;                // 1 .. 2^24-1
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

// Philox4x32-10 (bdm_internal.cuh) with the round keys precomputed on the host: they
// enter the XORs as constant-bank operands instead of two adds per round
__device__ __forceinline__ U4 philox10_rk(const SirArgs &A, uint32_t c0, uint32_t c1, uint32_t c2,
                                         uint32_t c3) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ A.rk0[r], n2 = hi0 ^ c3 ^ A.rk1[r];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return U4{c0, c1, c2, c3};
}

// Alg. 7/8 draws: uniform32(w) < p.  u = w 2^-32 is exact, so u < p <=> w < p 2^32 (exact
// scaling) <=> w < ceil(p 2^32): one integer comparison with the host's threshold
#ifndef BDM_SIR_INTCMP
#define BDM_SIR_INTCMP 1
#endif
__device__ __forceinline__ bool draw_below(uint32_t w, double p, unsigned long long t) {
#if BDM_SIR_INTCMP
    return (unsigned long long)w < t;
#else
    return uniform32(w) < p;
#endif
}
// Alg. 9's component 2 u - 1 with u = w 2^-32: 2u = w 2^-31 is exact, so the single
// rounding of fma(w, 2^-31, -1) is the rounding of 2u - 1 (bit-identical, no
// contraction of an inexact product)
#ifndef BDM_SIR_FMAV
#define BDM_SIR_FMAV 1
#endif
__device__ __forceinline__ double unit_comp(uint32_t w) {
#if BDM_SIR_FMAV
    return __fma_rn((double)w, 0x1p-31, -1.0);
#else
    return 2.0 * uniform32(w) - 1.0;
#endif
}

__device__ __forceinline__ double min_image(double d, double side, double half) {
    if (d > half) return d - side;
    if (d < -half) return d + side;
    return d;
}

__device__ void sir_insert(const SirArgs &A, int64_t i, DevScalars *__restrict__ sc);

// 16 states per thread (one 16-byte load when aligned); inserts the infected ones.
__global__ void __launch_bounds__(256) k_sir_collect(SirArgs A, DevScalars *__restrict__ sc) {
    const int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16;
    if (base >= A.n) return;
    if (base + 16 <= A.n && (((uintptr_t)(A.state + base)) & 15u) == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(A.state + base);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t x = w[q];
            // any byte == 1 (infected)?  (bytes are 0, 1 or 2)
            if (((x & 0x01010101u)) == 0u) continue;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (((x >> (8 * b)) & 0xFFu) == 1u) sir_insert(A, base + 4 * q + b, sc);
        }
    } else {
        for (int64_t i = base; i < A.n && i < base + 16; ++i)
            if (A.state[i] == 1) sir_insert(A, i, sc);
    }
}

__device__ void sir_insert(const SirArgs &A, int64_t i, DevScalars *__restrict__ sc) {
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
    const unsigned long long skey = (A.stamp << kStampShift) | key;
    unsigned long long h = box_hash(key, A.tbits);
    for (;;) {
        unsigned long long cur = A.keys[h];
        if (cur == skey) break;                       // box already present this step
        if ((cur >> kStampShift) != A.stamp) {        // stale slot: try to claim it
            const unsigned long long prev = atomicCAS(&A.keys[h], cur, skey);
            if (prev == cur || prev == skey) break;
            if ((prev >> kStampShift) != A.stamp) continue;  // lost to another stale write
        }
        h = (h + 1) & A.tmask;
    }
    const unsigned long long old = atomicExch(&A.heads[h], (A.stamp << 32) | slot);
    A.next[slot] = ((old >> 32) == A.stamp) ? (uint32_t)old : kNone;
    const uint32_t cb = (uint32_t)(((bz / A.cf) * A.B + (by / A.cf)) * A.B + (bx / A.cf));
    atomicOr(&A.bitmap[cb >> 5], 1u << (cb & 31u));
}

// Conservative coarse test: the coarse blocks (cf^3 fine boxes, edge C = cf L, cf = 16)
// that intersect [p - R', p + R'] per axis, R' = R(1 + 2^-20) + 2^-30 C, computed with
// a multiplication (no exactness needed: every fine box within R of p lies in one of
// them, since 2R' < C) and wrapped periodically by comparison.  D is a multiple of cf
// (the GPU's own fine lattice, L = side/D >= R), so every block is complete; for
// D < 32 a single block covers the space.
__device__ __forceinline__ int coarse_range(double p, double Rq, double invC, int B, int c[2]) {
    int lo = (int)floor((p - Rq) * invC), hi = (int)floor((p + Rq) * invC);
    lo = lo < 0 ? lo + B : (lo >= B ? lo - B : lo);
    hi = hi < 0 ? hi + B : (hi >= B ? hi - B : hi);
    c[0] = lo;
    c[1] = hi;
    return lo == hi ? 1 : 2;
}

__device__ __forceinline__ bool coarse_hit(const SirArgs &A, double px, double py, double pz) {
    int cx[2], cy[2], cz[2];
    const int nx = coarse_range(px, A.Rq, A.invC, A.B, cx);
    const int ny = coarse_range(py, A.Rq, A.invC, A.B, cy);
    const int nz = coarse_range(pz, A.Rq, A.invC, A.B, cz);
    bool hit = false;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (a < nz && b < ny && q < nx) {
                    const uint32_t cb = (uint32_t)((cz[a] * A.B + cy[b]) * A.B + cx[q]);
                    hit |= (A.bitmap[cb >> 5] >> (cb & 31u)) & 1u;
                }
            }
    return hit;
}

__device__ __forceinline__ bool infected_fine(const SirArgs &A, double px, double py, double pz);

__device__ __forceinline__ bool infected_within(const SirArgs &A, double px, double py, double pz) {
    if (!coarse_hit(A, px, py, pz)) return false;
    return infected_fine(A, px, py, pz);
}

// Exact search of the 27 fine boxes (same box formula as the index), minimum image.
__device__ __forceinline__ bool infected_fine(const SirArgs &A, double px, double py, double pz) {
    const int bx = sir_box(px, A.L, A.D), by = sir_box(py, A.L, A.D), bz = sir_box(pz, A.L, A.D);
    const int D = A.D;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int cx = bx + dx, cy = by + dy, cz = bz + dz;
                cx = cx < 0 ? cx + D : (cx >= D ? cx - D : cx);
                cy = cy < 0 ? cy + D : (cy >= D ? cy - D : cy);
                cz = cz < 0 ? cz + D : (cz >= D ? cz - D : cz);
                const unsigned long long key =
                    ((unsigned long long)cz * D + (unsigned long long)cy) * D + (unsigned long long)cx;
                const unsigned long long skey = (A.stamp << kStampShift) | key;
                unsigned long long h = box_hash(key, A.tbits);
                uint32_t head = kNone;
                for (;;) {
                    const unsigned long long k = A.keys[h];
                    if ((k >> kStampShift) != A.stamp) break;  // empty this step
                    if (k == skey) {
                        head = (uint32_t)A.heads[h];
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

// The IEEE quotient a / b from y = RN(1/b): q0 = RN(a y) is within one ulp of a / b,
// r = a - b q0 is exact (fma), and RN(q0 + r y) is the correctly rounded quotient
// (Markstein's theorem for a correctly rounded reciprocal, round to nearest, no
// overflow or underflow: here |a| <= 1 < b <= sqrt(3) and a is 0 or |a| >= 2^-31).
// Being correctly rounded, it equals a / b bit for bit; one IEEE division then serves
// the three components of the capped step (tests/test_gpu_sir.py checks it against a / b
// on 2^28 random operands, and every SIR parity test against the oracle's division).
__device__ __forceinline__ double div_by_recip(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q0, a);
    return __fma_rn(r, y, q0);
}

// Alg. 9 wrap: el = fmod(el, max); if el < 0: el = max + el (R20, literal).  For
// -max < el < 2 max, fmod is exact and equals el (|el| < max, sign kept: -0 stays -0 and
// is not < 0) or el - max (max <= el < 2 max, exact by Sterbenz), so the fast path is
// bit-identical to the literal form: el < 0 -> max + el, el >= max -> el - max, else el.
// fmod out of line: |el| >= max never happens in a unit-step walk, and an inlined fmod
// costs the whole kernel registers (spills): 1.94 -> 1.79 ms/step at cfg4
__device__ __noinline__ double fmod_slow(double el, double max_bound) { return fmod(el, max_bound); }
__device__ __forceinline__ double wrap_alg9(double el, double max_bound) {
    if (el > -max_bound && el < 2.0 * max_bound)
        return el < 0.0 ? max_bound + el : (el >= max_bound ? el - max_bound : el);
    const double r = fmod_slow(el, max_bound);
    return r < 0.0 ? max_bound + r : r;
}
__device__ __forceinline__ bool wrap_fast_ok(double el, double max_bound) {
    return el > -max_bound && el < 2.0 * max_bound;
}
// The fast path of wrap_alg9 as one subtraction: el - (-max) = max + el (the same IEEE
// sum), el - max, or el - 0 = el exactly (-0 stays -0)
__device__ __forceinline__ double wrap_fast(double el, double max_bound) {
    const double t = el < 0.0 ? -max_bound : (el >= max_bound ? max_bound : 0.0);
    return el - t;
}

// Infection queries (S agents whose draw passed, ~p_inf of them) are compacted into a
// per-warp queue with their start-of-step position and resolved 32 at a time, one per
// lane, so the index search does not run with a few lanes of each warp; movement and
// the other state updates do not depend on the query and proceed at once.
constexpr int kSirThreads = 256;
constexpr int kSirQ = 64;  // queue entries per warp (<= 31 left over + <= 32 new)

struct SirQueue {
    uint32_t idx[kSirQ];
    double px[kSirQ], py[kSirQ], pz[kSirQ];
};

// Per-thread S/I/R counts of the final states.  Packed: one 64-bit add per agent,
// S | I << 21 | R << 42 (a thread counts fewer than 2^21 agents; launch_sir_step checks
// the bound)
#ifndef BDM_SIR_PACKED
#define BDM_SIR_PACKED 1
#endif
struct SirCnt {
#if BDM_SIR_PACKED
    unsigned long long pk = 0;
    __device__ __forceinline__ void add(uint32_t st) { pk += 1ull << (21u * st); }
    __device__ __forceinline__ uint32_t s() const { return (uint32_t)(pk & 0x1FFFFFull); }
    __device__ __forceinline__ uint32_t i() const { return (uint32_t)((pk >> 21) & 0x1FFFFFull); }
    __device__ __forceinline__ uint32_t r() const { return (uint32_t)(pk >> 42); }
#else
    uint32_t cs = 0, ci = 0, cr = 0;
    __device__ __forceinline__ void add(uint32_t st) {
        cs += st == 0;
        ci += st == 1;
        cr += st == 2;
    }
    __device__ __forceinline__ uint32_t s() const { return cs; }
    __device__ __forceinline__ uint32_t i() const { return ci; }
    __device__ __forceinline__ uint32_t r() const { return cr; }
#endif
};

// The final state of a queried S agent and its counters.
__device__ __forceinline__ void sir_resolve(const SirArgs &A, uint32_t i, double px, double py,
                                            double pz, SirCnt &cc,
                                            uint32_t &cn) {
    uint8_t st = 0;
    if (infected_within(A, px, py, pz)) {
        st = 1;
        ++cn;
        const uint32_t me = A.id ? A.id[i] : i;
        const U4 r = philox10_rk(A, me, 0u, A.step, 1u);
        if (draw_below(r.a, A.p_rec, A.t_rec)) st = 2;  // Alg. 8 in sequence (R18)
    }
    A.state[i] = st;
    cc.add(st);
}

// Whether box (bx+dx, by+dy, bz+dz) (periodic) holds a snapshot-I agent within R of p
// (minimum image): the same box formula, key, hash probe and chain walk as
// infected_fine, for one box.
__device__ __forceinline__ bool infected_in_box(const SirArgs &A, double px, double py, double pz, int bx,
                                                int by, int bz, int dx, int dy, int dz) {
    const int D = A.D;
    int cx = bx + dx, cy = by + dy, cz = bz + dz;
    cx = cx < 0 ? cx + D : (cx >= D ? cx - D : cx);
    cy = cy < 0 ? cy + D : (cy >= D ? cy - D : cy);
    cz = cz < 0 ? cz + D : (cz >= D ? cz - D : cz);
    const unsigned long long key =
        ((unsigned long long)cz * D + (unsigned long long)cy) * D + (unsigned long long)cx;
    const unsigned long long skey = (A.stamp << kStampShift) | key;
    unsigned long long h = box_hash(key, A.tbits);
    uint32_t head = kNone;
    for (;;) {
        const unsigned long long k = A.keys[h];
        if ((k >> kStampShift) != A.stamp) break;  // empty this step
        if (k == skey) {
            head = (uint32_t)A.heads[h];
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
    return false;
}

// The queued queries Q[0, nq) of a warp (nq <= 32, warp-uniform), one per lane: the
// coarse test per lane, then each query that passes it is searched by the whole warp,
// lane b < 27 taking box b of the 27 (their hash probes and chains in parallel instead
// of one lane walking all 27 boxes while the others wait).  "Any snapshot-I agent within
// R" does not depend on the order of the boxes, so the result is the same.
__device__ __forceinline__ void sir_resolve_warp(const SirArgs &A, const SirQueue &Q, int lane, int nq,
                                                 SirCnt &cc, uint32_t &cn) {
    const bool act = lane < nq;
    uint32_t i = 0;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (act) {
        i = Q.idx[lane];
        px = Q.px[lane];
        py = Q.py[lane];
        pz = Q.pz[lane];
    }
    unsigned hm = __ballot_sync(0xffffffffu, act && coarse_hit(A, px, py, pz));
    bool inf = false;
    const int ddx = lane % 3 - 1, ddy = (lane / 3) % 3 - 1, ddz = lane / 9 - 1;
    while (hm) {  // warp-uniform
        const int q = __ffs(hm) - 1;
        hm &= hm - 1;
        const double qx = __shfl_sync(0xffffffffu, px, q), qy = __shfl_sync(0xffffffffu, py, q),
                     qz = __shfl_sync(0xffffffffu, pz, q);
        bool found = false;
        if (lane < 27) {
            const int bx = sir_box(qx, A.L, A.D), by = sir_box(qy, A.L, A.D), bz = sir_box(qz, A.L, A.D);
            found = infected_in_box(A, qx, qy, qz, bx, by, bz, ddx, ddy, ddz);
        }
        const bool any = __any_sync(0xffffffffu, found);
        if (lane == q) inf = any;
    }
    if (act) {
        uint8_t st = 0;
        if (inf) {
            st = 1;
            ++cn;
            const uint32_t me = A.id ? A.id[i] : i;
            const U4 r = philox10_rk(A, me, 0u, A.step, 1u);
            if (draw_below(r.a, A.p_rec, A.t_rec)) st = 2;  // Alg. 8 in sequence (R18)
        }
        A.state[i] = st;
        cc.add(st);
    }
}

// One agent of the update (its start-of-step x, y, z, state already loaded): Philox
// draws, the queue entry for an infection query, recovery, movement and wrap.
template <typename I>
__device__ __forceinline__ void sir_agent(const SirArgs &A, SirQueue &Q, int lane, unsigned lt_mask,
                                          I i, bool valid, double px, double py, double pz,
                                          uint8_t st, uint32_t me, int &qn, SirCnt &cc, uint32_t &cn) {
    const U4 w = philox10_rk(A, me, 0u, A.step, 0u);
    // Alg. 7: an S agent whose draw passed (R17: strict '<', u = w * 2^-32) is queued
    const bool query = valid && st == 0 && draw_below(w.d, A.p_inf, A.t_inf);
    if (valid && !query) {
        // Alg. 8: recovery (own state in sequence, R18)
        if (st == 1) {
            const U4 r = philox10_rk(A, me, 0u, A.step, 1u);
            if (draw_below(r.a, A.p_rec, A.t_rec)) {
                st = 2;
                A.state[i] = st;
            }
        }
        cc.add(st);
    }
    // Alg. 9: movement capped at unit length (R16), toroidal wrap (R20)
    if (valid) {
        double vx = unit_comp(w.a);
        double vy = unit_comp(w.b);
        double vz = unit_comp(w.c);
        const double v2 = vx * vx + vy * vy + vz * vz;
        {  // straight-line: 48 % of the lanes need the cap, the warp runs it anyway
            const double nv = sqrt(v2);
            const bool cap = v2 > 1.0;
#ifndef BDM_SIR_DIV3
            // the three IEEE quotients v/nv share one reciprocal (div_by_recip)
            const double rn = 1.0 / nv;
            const double qx = div_by_recip(vx, nv, rn), qy = div_by_recip(vy, nv, rn),
                         qz = div_by_recip(vz, nv, rn);
#else
            const double qx = vx / nv, qy = vy / nv, qz = vz / nv;
#endif
            vx = cap ? qx : vx;
            vy = cap ? qy : vy;
            vz = cap ? qz : vz;
        }
#ifndef BDM_SIR_OLDWRAP
        // one range test for the three coordinates (the literal fmod form only off it)
        const double ex = px + vx, ey = py + vy, ez = pz + vz;
        if (wrap_fast_ok(ex, A.side) && wrap_fast_ok(ey, A.side) && wrap_fast_ok(ez, A.side)) {
            A.x[i] = wrap_fast(ex, A.side);
            A.y[i] = wrap_fast(ey, A.side);
            A.z[i] = wrap_fast(ez, A.side);
        } else {
            A.x[i] = wrap_alg9(ex, A.side);
            A.y[i] = wrap_alg9(ey, A.side);
            A.z[i] = wrap_alg9(ez, A.side);
        }
#else
        A.x[i] = wrap_alg9(px + vx, A.side);
        A.y[i] = wrap_alg9(py + vy, A.side);
        A.z[i] = wrap_alg9(pz + vz, A.side);
#endif
    }
    // queue the infection queries (start-of-step positions)
    const unsigned qb = __ballot_sync(0xffffffffu, query);
    if (query) {
        const int p = qn + __popc(qb & lt_mask);
        Q.idx[p] = (uint32_t)i;
        Q.px[p] = px;
        Q.py[p] = py;
        Q.pz[p] = pz;
    }
    qn += __popc(qb);
    if (qn >= 32) {  // warp-uniform: resolve 32 queries, one per lane
        __syncwarp();
#ifdef BDM_SIR_LANE_SEARCH
        sir_resolve(A, Q.idx[lane], Q.px[lane], Q.py[lane], Q.pz[lane], cc, cn);
#else
        sir_resolve_warp(A, Q, lane, 32, cc, cn);
#endif
        __syncwarp();
        qn -= 32;
        if (lane < qn) {
            Q.idx[lane] = Q.idx[32 + lane];
            Q.px[lane] = Q.px[32 + lane];
            Q.py[lane] = Q.py[32 + lane];
            Q.pz[lane] = Q.pz[32 + lane];
        }
        __syncwarp();
    }
}

#ifndef BDM_SIR_MINB
#define BDM_SIR_MINB 4  // resident blocks per SM the register budget is set for
#endif
#ifndef BDM_SIR_IDPF
#define BDM_SIR_IDPF 0
#endif
// I: the agent index type, uint32_t when n + the grid stride < 2^32 (32-bit address
// arithmetic; the queue holds 32-bit indices in either case), else int64_t
template <typename I>
__global__ void __launch_bounds__(kSirThreads, BDM_SIR_MINB) k_sir_update(SirArgs A, DevScalars *__restrict__ sc) {
    if (sc->overflow) return;
    __shared__ SirQueue Qs[kSirThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    SirQueue &Q = Qs[wid];
    const unsigned lt_mask = (1u << lane) - 1u;
    // per-thread counters: a thread sees at most n / (grid threads) agents (< 2^32)
    SirCnt cc;
    uint32_t cn = 0;
    int qn = 0;  // warp-uniform queue fill
    const I nwarps = (I)gridDim.x * (I)(kSirThreads / 32);
    const I first = ((I)blockIdx.x * (I)(kSirThreads / 32) + (I)wid) * (I)64, stride = nwarps * (I)64;
    const I n = (I)A.n;
    // two 32-agent slices per warp iteration, all their loads issued first (staging
    // the next 64 agents in shared memory with cp.async while computing measured
    // slower: 1.62 vs 1.58 ms at cfg4)
#if BDM_SIR_IDPF
    // the ids (Philox counters) are loaded one iteration ahead: the first Philox round of
    // an iteration no longer waits on this iteration's loads
    uint32_t na = 0, nb = 0;
    {
        const I ia = first + (I)lane, ib = first + (I)(32 + lane);
        if (ia < n) na = A.id ? A.id[ia] : (uint32_t)ia;
        if (ib < n) nb = A.id ? A.id[ib] : (uint32_t)ib;
    }
#endif
    for (I i0 = first; i0 < n; i0 += stride) {
        const I ia = i0 + (I)lane, ib = i0 + (I)(32 + lane);
        const bool va = ia < n, vb = ib < n;
        double xa = 0.0, ya = 0.0, za = 0.0, xb = 0.0, yb = 0.0, zb = 0.0;
        uint8_t sa = 0, sb = 0;
#if BDM_SIR_IDPF
        const uint32_t ma = na, mb = nb;
        {
            const I ja = ia + stride, jb = ib + stride;
            if (ja < n) na = A.id ? A.id[ja] : (uint32_t)ja;
            if (jb < n) nb = A.id ? A.id[jb] : (uint32_t)jb;
        }
        if (va) {
            xa = A.x[ia];
            ya = A.y[ia];
            za = A.z[ia];
            sa = A.state[ia];
        }
        if (vb) {
            xb = A.x[ib];
            yb = A.y[ib];
            zb = A.z[ib];
            sb = A.state[ib];
        }
#else
        uint32_t ma = 0, mb = 0;  // ids (Philox counters), loaded with the rest
        if (va) {
            xa = A.x[ia];
            ya = A.y[ia];
            za = A.z[ia];
            sa = A.state[ia];
            ma = A.id ? A.id[ia] : (uint32_t)ia;
        }
        if (vb) {
            xb = A.x[ib];
            yb = A.y[ib];
            zb = A.z[ib];
            sb = A.state[ib];
            mb = A.id ? A.id[ib] : (uint32_t)ib;
        }
#endif
        sir_agent(A, Q, lane, lt_mask, ia, va, xa, ya, za, sa, ma, qn, cc, cn);
        sir_agent(A, Q, lane, lt_mask, ib, vb, xb, yb, zb, sb, mb, qn, cc, cn);
    }
    __syncwarp();
#ifdef BDM_SIR_LANE_SEARCH
    if (lane < qn) sir_resolve(A, Q.idx[lane], Q.px[lane], Q.py[lane], Q.pz[lane], cc, cn);
#else
    sir_resolve_warp(A, Q, lane, qn, cc, cn);
#endif
    // block reduction of the counters, one atomic each per block
    __shared__ unsigned long long red[4][kSirThreads / 32];
    unsigned long long v[4] = {cc.s(), cc.i(), cc.r(), cn};  // warp sums in 64 bits
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
        for (int k = 0; k < kSirThreads / 32; ++k) t += red[threadIdx.x][k];
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
    // the hash key packs the box index below the step stamp (kStampShift = 40 bits), so
    // D^3 must stay below 2^40: D <= 8192 boxes per axis (checked before the int cast)
    const double ratio = side / radius;
    if (!(ratio >= 3.0) || !(ratio < 8193.0)) {
        set_error("SIR needs 3 <= side / radius < 8193 (boxes per axis; the infected-index "
                  "hash keys hold D^3 < 2^40)");
        return BDM_EINVAL;
    }
    const int D0 = (int)floor(ratio);
    // the GPU's fine lattice: L = side/D >= R, D a multiple of kCoarse when large (the
    // box size does not enter any result: the infection test is exact for any L >= R)
    const int D = D0 >= 2 * kCoarse ? D0 - D0 % kCoarse : D0;
    const int cf = D0 >= 2 * kCoarse ? kCoarse : (D0 > 0 ? D0 : 1);
    if (D < 3) {
        set_error("SIR needs side / radius >= 3 boxes per axis");
        return BDM_EINVAL;
    }
    if ((long long)D * D * D >= (1ll << kStampShift)) {
        set_error("SIR grid too large (D^3 >= 2^40)");
        return BDM_EINVAL;
    }
    const int B = D / cf;
    const int64_t want_icap = a->n / 16 > 65536 ? a->n / 16 : 65536;
    const int64_t icap = W.icap_override > 0 ? W.icap_override : want_icap;
    const int tbits = next_pow2_bits(2 * icap);
    const int64_t tsize = 1ll << tbits;
    const int64_t bwords = ((int64_t)B * B * B + 31) / 32;
    if (icap > W.icap || tsize > W.tsize || bwords > W.bwords) {
        BDM_CUDA_TRY(cudaStreamSynchronize(st));
        void *old[] = {W.keys, W.heads, W.next, W.ix, W.iy, W.iz, W.bitmap, W.misc};
        for (void *q : old)
            if (q) cudaFree(q);
        W = SirWs{};
        if (cudaMalloc(&W.keys, tsize * 8) != cudaSuccess ||
            cudaMalloc(&W.heads, tsize * 8) != cudaSuccess ||
            cudaMalloc(&W.next, icap * 4) != cudaSuccess || cudaMalloc(&W.ix, icap * 8) != cudaSuccess ||
            cudaMalloc(&W.iy, icap * 8) != cudaSuccess || cudaMalloc(&W.iz, icap * 8) != cudaSuccess ||
            cudaMalloc(&W.bitmap, bwords * 4) != cudaSuccess ||
            cudaMalloc(&W.misc, 64) != cudaSuccess) {
            cudaGetLastError();
            set_error("SIR workspace allocation failed");
            return BDM_ECAPACITY;
        }
        W.icap = icap;
        W.tsize = tsize;
        W.bwords = bwords;
        // fresh table: stamp 0 marks every slot empty
        BDM_CUDA_TRY(cudaMemsetAsync(W.keys, 0, tsize * 8, st));
        BDM_CUDA_TRY(cudaMemsetAsync(W.heads, 0, tsize * 8, st));
        W.stamp = 0;
    }
    if (++W.stamp >= (1ull << 24)) {  // stamp wrap: clear once and restart
        BDM_CUDA_TRY(cudaMemsetAsync(W.keys, 0, W.tsize * 8, st));
        BDM_CUDA_TRY(cudaMemsetAsync(W.heads, 0, W.tsize * 8, st));
        W.stamp = 1;
    }
    if (!W.misc) BDM_CUDA_TRY(cudaMalloc(&W.misc, 64));
    SirArgs A;
    A.n = a->n;
    A.x = a->x; A.y = a->y; A.z = a->z; A.state = a->state; A.id = a->id;
    A.side = side;
    A.L = side / (double)D;
    A.cf = cf;
    A.invC = 1.0 / (A.L * (double)cf);
    A.Rq = radius * (1.0 + 0x1p-20) + A.L * (double)cf * 0x1p-30;
    A.R2 = radius * radius;
    A.half = side * 0.5;
    A.p_inf = p_inf;
    A.p_rec = p_rec;
    {
        auto thr = [](double q) -> unsigned long long {
            const double sc = q * 4294967296.0;  // exact (power-of-two scaling)
            if (!(sc > 0.0)) return 0ull;        // never (incl. NaN: u < NaN is false)
            if (sc >= 4294967296.0) return 4294967296ull;  // always
            return (unsigned long long)ceil(sc);
        };
        A.t_inf = thr(p_inf);
        A.t_rec = thr(p_rec);
    }
    A.D = D;
    A.B = B;
    A.k0 = (uint32_t)p->seed;
    A.k1 = (uint32_t)(p->seed >> 32);
    for (int r = 0; r < 10; ++r) {
        A.rk0[r] = A.k0 + 0x9E3779B9u * (uint32_t)r;
        A.rk1[r] = A.k1 + 0xBB67AE85u * (uint32_t)r;
    }
    A.step = p->step;
    A.keys = W.keys; A.heads = (unsigned long long *)W.heads; A.next = W.next;
    A.stamp = W.stamp;
    A.ix = W.ix; A.iy = W.iy; A.iz = W.iz;
    A.bitmap = W.bitmap;
    A.icount = (uint32_t *)W.misc;
    A.counts = (unsigned long long *)((char *)W.misc + 32);
    A.icap = (uint32_t)W.icap;
    A.tbits = tbits;
    A.tmask = (unsigned long long)(tsize - 1);
    BDM_CUDA_TRY(cudaMemsetAsync(W.bitmap, 0, ((int64_t)B * B * B + 31) / 32 * 4, st));
    BDM_CUDA_TRY(cudaMemsetAsync(W.misc, 0, 64, st));
    if (a->n > 0) {
        int64_t ub = (a->n + 255) / 256;
        // one resident wave (4 blocks per SM, the launch bounds) striding over the
        // agents: no partial last wave (1.99 -> 1.96 ms/step at cfg4)
        const int64_t maxb = (int64_t)c->sm_count * 4;
        if (ub > maxb) ub = maxb;
        // packed per-thread S/I/R counts (SirCnt): at most 4 ceil(n / threads) per thread
        if (4 * ((a->n + ub * kSirThreads - 1) / (ub * kSirThreads)) >= (1ll << 21)) {
            set_error("SIR population too large for the per-thread counters of this GPU");
            return BDM_EINVAL;
        }
        const unsigned nb = (unsigned)(((a->n + 15) / 16 + 255) / 256);
        k_sir_collect<<<nb, 256, 0, st>>>(A, c->sc);
#ifndef BDM_SIR_FORCE64
#define BDM_SIR_FORCE64 0
#endif
        if (!BDM_SIR_FORCE64 && a->n + ub * kSirThreads * 2 < (1ll << 32))
            k_sir_update<uint32_t><<<(unsigned)ub, kSirThreads, 0, st>>>(A, c->sc);
        else
            k_sir_update<int64_t><<<(unsigned)ub, kSirThreads, 0, st>>>(A, c->sc);
        c->launches += 2;
        BDM_LAUNCH_CHECK("SIR kernels");
    }
    if (counts_host)
        BDM_CUDA_TRY(cudaMemcpyAsync(counts_host, A.counts, 4 * sizeof(long long),
                                     cudaMemcpyDeviceToHost, st));
    return BDM_OK;
}

// ---- self-test of div_by_recip against IEEE division (bdm_selftest_recip_div)
__global__ void k_selftest_recip_div(int64_t n, uint32_t k0, uint32_t k1, unsigned long long *bad) {
    unsigned long long nb = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const U4 w = philox10((uint32_t)i, (uint32_t)(i >> 32), 0x5eedu, 7u, k0, k1);
        const double vx = 2.0 * uniform32(w.a) - 1.0, vy = 2.0 * uniform32(w.b) - 1.0,
                     vz = 2.0 * uniform32(w.c) - 1.0;
        const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        if (!(v2 > 1.0)) continue;
        const double nv = sqrt(v2), rn = 1.0 / nv;
        nb += __double_as_longlong(div_by_recip(vx, nv, rn)) != __double_as_longlong(vx / nv);
        nb += __double_as_longlong(div_by_recip(vy, nv, rn)) != __double_as_longlong(vy / nv);
        nb += __double_as_longlong(div_by_recip(vz, nv, rn)) != __double_as_longlong(vz / nv);
    }
    if (nb) atomicAdd(bad, nb);
}

bdm_status launch_selftest_recip_div(Ctx *c, int64_t n, uint64_t seed, unsigned long long *mismatches) {
    unsigned long long *d = nullptr;
    BDM_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long)));
    BDM_CUDA_TRY(cudaMemset(d, 0, sizeof(unsigned long long)));
    k_selftest_recip_div<<<(unsigned)(c->sm_count * 8), 256>>>(n, (uint32_t)seed, (uint32_t)(seed >> 32), d);
    const cudaError_t e = cudaMemcpy(mismatches, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    BDM_CUDA_TRY(e);
    return BDM_OK;
}

}  // namespace bdm
