// mech_common.cuh -- pieces shared by the mechanics kernels (kernels_mech.cu: the
// reference, tile and dense-box kernels; kernels_row.cu: the row-broadcast kernel):
// kernel arguments, the grid scalars, per-agent counters, the a8/a9 epilogue and the
// reference formulation of the whole step for one agent.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

struct MechArgs {
    int64_t n;
    const double *__restrict__ sx;
    const double *__restrict__ sy;
    const double *__restrict__ sz;
    const double *__restrict__ sd;
    const uint32_t *__restrict__ sid;
    const uint32_t *__restrict__ skey;  // sorted blocked-Morton key (box of each sorted slot)
    const uint32_t *__restrict__ sflags;
    const uint32_t *__restrict__ box_start;
    double *__restrict__ ox;
    double *__restrict__ oy;
    double *__restrict__ oz;
    double *__restrict__ od;
    uint32_t *__restrict__ oid;
    uint32_t *__restrict__ oflags;
    const uint32_t *__restrict__ lrank;  // nullable: output index of sorted local slots (ghosts)
    const double *__restrict__ svol;  // nullable: volume travels with the agents
    double *__restrict__ ovol;
    uint32_t *__restrict__ dense_list;   // nullable: dense tiles go to k_mech_dense
    uint32_t *__restrict__ dense_perm;   // dense kernel: kDScr entries of scratch per warp
    double k, gamma, dt, max_disp, tau;
    int detect_static, boundary, fuse;
    double lo0, lo1, lo2, hi0, hi1, hi2;
};

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Grid scalars of the current step, read once per thread/CTA.
struct GridView {
    double L, R2, o0, o1, o2;
    int D0, D1, D2, T0, T1, T2;
    int b0, b1, b2;  // lattice offset (global frame, 8(e))
    const uint16_t *hilb, *hilb_inv;  // tile numbering (NULL: row-major)
};
__device__ __forceinline__ GridView load_grid(const DevScalars *__restrict__ sc) {
    GridView g;
    g.L = sc->L; g.R2 = sc->R2; g.o0 = sc->o[0]; g.o1 = sc->o[1]; g.o2 = sc->o[2];
    g.b0 = sc->boff[0]; g.b1 = sc->boff[1]; g.b2 = sc->boff[2];
    g.D0 = sc->dims[0]; g.D1 = sc->dims[1]; g.D2 = sc->dims[2];
    g.T0 = sc->T[0]; g.T1 = sc->T[1]; g.T2 = sc->T[2];
    g.hilb = sc_hilb(sc);
    g.hilb_inv = sc_hilb_inv(sc);
    return g;
}

struct Counts {
    uint32_t cand = 0, nbr = 0, cont = 0, stat = 0, moved = 0;
    // extent of the new state (a1 of the next step, fused: option "fuse_reduce")
    double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY;
    double hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY, dmax = -INFINITY;
};

// a8 + a9 + write-back for one agent (shared by both kernels); s is the sorted slot,
// the output goes to lrank[s] when ghosts are present.  di and idi are the agent's
// diameter and id (the tile kernels have them in registers before the step's work).
__device__ __forceinline__ void finish_agent(const MechArgs &A, int64_t s, double xi, double yi,
                                             double zi, double Fx, double Fy, double Fz,
                                             bool is_static, int nnz, Counts &c, bool track,
                                             double di, uint32_t idi) {
    const int64_t o = A.lrank ? (int64_t)A.lrank[s] : s;
    double Dx = 0.0, Dy = 0.0, Dz = 0.0;
    if (!is_static) {
        const double F2 = Fx * Fx + Fy * Fy + Fz * Fz;
        if (F2 > A.tau * A.tau) {
            Dx = A.dt * Fx;
            Dy = A.dt * Fy;
            Dz = A.dt * Fz;
            const double n2 = Dx * Dx + Dy * Dy + Dz * Dz;
            if (n2 > A.max_disp * A.max_disp) {
                const double scale = A.max_disp / sqrt(n2);
                Dx = Dx * scale;
                Dy = Dy * scale;
                Dz = Dz * scale;
            }
        }
    }
    double nx = xi + Dx, ny = yi + Dy, nz = zi + Dz;
    if (A.boundary == 1) {
        nx = nx < A.lo0 ? A.lo0 : (nx > A.hi0 ? A.hi0 : nx);
        ny = ny < A.lo1 ? A.lo1 : (ny > A.hi1 ? A.hi1 : ny);
        nz = nz < A.lo2 ? A.lo2 : (nz > A.hi2 ? A.hi2 : nz);
    } else if (A.boundary == 2) {  // toroidal [0, hi0)^3: Alg. 9's literal wrap (R20, R52)
        double r = fmod(nx, A.hi0);
        nx = r < 0.0 ? A.hi0 + r : r;
        r = fmod(ny, A.hi0);
        ny = r < 0.0 ? A.hi0 + r : r;
        r = fmod(nz, A.hi0);
        nz = r < 0.0 ? A.hi0 + r : r;
    }
    const bool moved = (Dx != 0.0 || Dy != 0.0 || Dz != 0.0);
    c.moved += moved ? 1u : 0u;
    if (track) {  // (the tile kernels skip it where no extremum can move, see k_mech_tile6)
        c.lo0 = fmin(c.lo0, nx); c.hi0 = fmax(c.hi0, nx);
        c.lo1 = fmin(c.lo1, ny); c.hi1 = fmax(c.hi1, ny);
        c.lo2 = fmin(c.lo2, nz); c.hi2 = fmax(c.hi2, nz);
        c.dmax = fmax(c.dmax, di);
    }
    c.stat += is_static ? 1u : 0u;
    A.ox[o] = nx;
    A.oy[o] = ny;
    A.oz[o] = nz;
    A.od[o] = di;
    A.oid[o] = idi;
    if (A.ovol) A.ovol[o] = A.svol[s];
    A.oflags[o] = (moved ? BDM_FLAG_MOVED : 0u) | (is_static ? BDM_FLAG_STATIC : 0u) |
                  ((uint32_t)nnz << BDM_FLAG_NNZ_SHIFT);
}

__device__ __forceinline__ void finish_agent(const MechArgs &A, int64_t s, double xi, double yi,
                                             double zi, double Fx, double Fy, double Fz,
                                             bool is_static, int nnz, Counts &c,
                                             bool track = true) {
    finish_agent(A, s, xi, yi, zi, Fx, Fy, Fz, is_static, nnz, c, track, A.sd[s], A.sid[s]);
}

// The whole step for agent s of the sorted order, reading neighbours from global
// memory (the reference formulation; used by k_mech and as the tile kernel's
// fallback for over-full tiles).
__device__ __forceinline__ void mech_agent_global(const MechArgs &A, const GridView &g, int64_t s,
                                                  Counts &c) {
    const uint32_t fi = A.sflags[s];
    if (fi & kGhost) return;  // aura agents are read-only
    const double xi = A.sx[s], yi = A.sy[s], zi = A.sz[s], di = A.sd[s];
    const double ri = di * 0.5;
    const int bx = (int)floor((xi - g.o0) / g.L) - g.b0;
    const int by = (int)floor((yi - g.o1) / g.L) - g.b1;
    const int bz = (int)floor((zi - g.o2) / g.L) - g.b2;
    const int nnz_in = (int)((fi >> BDM_FLAG_NNZ_SHIFT) & 3u);

    // ---- a5: static classification (pull test over the neighbours' flags)
    bool is_static = false;
    if (A.detect_static && !(fi & kChanged) && nnz_in <= 1) {
        is_static = true;
        for (int dz = -1; dz <= 1 && is_static; ++dz) {
            const int cz = bz + dz;
            if (cz < 0 || cz >= g.D2) continue;
            for (int dy = -1; dy <= 1 && is_static; ++dy) {
                const int cy = by + dy;
                if (cy < 0 || cy >= g.D1) continue;
                for (int dx = -1; dx <= 1 && is_static; ++dx) {
                    const int cx = bx + dx;
                    if (cx < 0 || cx >= g.D0) continue;
                    const uint32_t key = box_key(cx, cy, cz, g.T0, g.T1, g.hilb);
                    const uint32_t b0 = A.box_start[key], b1 = A.box_start[key + 1];
                    for (uint32_t t = b0; t < b1; ++t) {
                        if (t == (uint32_t)s) continue;
                        const double ex = xi - A.sx[t], ey = yi - A.sy[t], ez = zi - A.sz[t];
                        const double D = fma(ez, ez, fma(ey, ey, ex * ex));
                        if (D <= g.R2 && (A.sflags[t] & kChanged)) {
                            is_static = false;
                            break;
                        }
                    }
                }
            }
        }
    }
    double Fx = 0.0, Fy = 0.0, Fz = 0.0;
    int nnz = nnz_in;
    if (!is_static) {
        // ---- a6 + a7: canonical order (dz, dy, dx), ascending id in a box
        nnz = 0;
        for (int dz = -1; dz <= 1; ++dz) {
            const int cz = bz + dz;
            if (cz < 0 || cz >= g.D2) continue;
            for (int dy = -1; dy <= 1; ++dy) {
                const int cy = by + dy;
                if (cy < 0 || cy >= g.D1) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    const int cx = bx + dx;
                    if (cx < 0 || cx >= g.D0) continue;
                    const uint32_t key = box_key(cx, cy, cz, g.T0, g.T1, g.hilb);
                    const uint32_t b0 = A.box_start[key], b1 = A.box_start[key + 1];
                    for (uint32_t t = b0; t < b1; ++t) {
                        if (t == (uint32_t)s) continue;
                        ++c.cand;
                        const double ex = xi - A.sx[t], ey = yi - A.sy[t], ez = zi - A.sz[t];
                        const double D = fma(ez, ez, fma(ey, ey, ex * ex));
                        if (!(D <= g.R2)) continue;
                        ++c.nbr;
                        const double dist = sqrt(D);
                        const double rj = A.sd[t] * 0.5;
                        const double delta = (ri + rj) - dist;
                        if (!(delta > 0.0 && dist > 0.0)) continue;
                        ++c.cont;
                        const double rbar = (ri * rj) / (ri + rj);
                        const double Fn = A.k * delta - A.gamma * sqrt(rbar * delta);
                        const double sc_ = Fn / dist;
                        Fx = fma(sc_, ex, Fx);
                        Fy = fma(sc_, ey, Fy);
                        Fz = fma(sc_, ez, Fz);
                        if (Fn != 0.0 && nnz < 2) ++nnz;
                    }
                }
            }
        }
    }
    finish_agent(A, s, xi, yi, zi, Fx, Fy, Fz, is_static, nnz, c);
}

// Toroidal mechanics (boundary 2, R52) for agent s: the reference formulation on the
// periodic lattice of [0, side)^3 -- the 27 boxes wrap modulo D in canonical order
// (dz, dy, dx), ascending id in a box (R9); every difference is the minimum image
// (own - other, +-side beyond side/2) before D and f_ij.
__device__ __forceinline__ double torus_image(double v, double side, double half) {
    return v > half ? v - side : (v < -half ? v + side : v);
}
__device__ __forceinline__ int torus_wrap(int c, int D) { return c < 0 ? c + D : (c >= D ? c - D : c); }
__device__ __forceinline__ void mech_agent_torus(const MechArgs &A, const GridView &g, int64_t s,
                                                 double side, Counts &c) {
    const uint32_t fi = A.sflags[s];
    if (fi & kGhost) return;
    const double half = side * 0.5;
    const double xi = A.sx[s], yi = A.sy[s], zi = A.sz[s], di = A.sd[s];
    const double ri = di * 0.5;
    int bx = (int)floor(xi / g.L), by = (int)floor(yi / g.L), bz = (int)floor(zi / g.L);
    bx = bx < 0 ? 0 : (bx > g.D0 - 1 ? g.D0 - 1 : bx);
    by = by < 0 ? 0 : (by > g.D1 - 1 ? g.D1 - 1 : by);
    bz = bz < 0 ? 0 : (bz > g.D2 - 1 ? g.D2 - 1 : bz);
    const int nnz_in = (int)((fi >> BDM_FLAG_NNZ_SHIFT) & 3u);
    bool is_static = false;
    if (A.detect_static && !(fi & kChanged) && nnz_in <= 1) {
        is_static = true;
        for (int dz = -1; dz <= 1 && is_static; ++dz)
            for (int dy = -1; dy <= 1 && is_static; ++dy)
                for (int dx = -1; dx <= 1 && is_static; ++dx) {
                    const uint32_t key = box_key(torus_wrap(bx + dx, g.D0), torus_wrap(by + dy, g.D1),
                                                 torus_wrap(bz + dz, g.D2), g.T0, g.T1, g.hilb);
                    const uint32_t b0 = A.box_start[key], b1 = A.box_start[key + 1];
                    for (uint32_t t = b0; t < b1; ++t) {
                        if (t == (uint32_t)s) continue;
                        const double ex = torus_image(xi - A.sx[t], side, half);
                        const double ey = torus_image(yi - A.sy[t], side, half);
                        const double ez = torus_image(zi - A.sz[t], side, half);
                        const double D = fma(ez, ez, fma(ey, ey, ex * ex));
                        if (D <= g.R2 && (A.sflags[t] & kChanged)) {
                            is_static = false;
                            break;
                        }
                    }
                }
    }
    double Fx = 0.0, Fy = 0.0, Fz = 0.0;
    int nnz = nnz_in;
    if (!is_static) {
        nnz = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const uint32_t key = box_key(torus_wrap(bx + dx, g.D0), torus_wrap(by + dy, g.D1),
                                                 torus_wrap(bz + dz, g.D2), g.T0, g.T1, g.hilb);
                    const uint32_t b0 = A.box_start[key], b1 = A.box_start[key + 1];
                    for (uint32_t t = b0; t < b1; ++t) {
                        if (t == (uint32_t)s) continue;
                        ++c.cand;
                        const double ex = torus_image(xi - A.sx[t], side, half);
                        const double ey = torus_image(yi - A.sy[t], side, half);
                        const double ez = torus_image(zi - A.sz[t], side, half);
                        const double D = fma(ez, ez, fma(ey, ey, ex * ex));
                        if (!(D <= g.R2)) continue;
                        ++c.nbr;
                        const double dist = sqrt(D);
                        const double rj = A.sd[t] * 0.5;
                        const double delta = (ri + rj) - dist;
                        if (!(delta > 0.0 && dist > 0.0)) continue;
                        ++c.cont;
                        const double rbar = (ri * rj) / (ri + rj);
                        const double Fn = A.k * delta - A.gamma * sqrt(rbar * delta);
                        const double sc_ = Fn / dist;
                        Fx = fma(sc_, ex, Fx);
                        Fy = fma(sc_, ey, Fy);
                        Fz = fma(sc_, ez, Fz);
                        if (Fn != 0.0 && nnz < 2) ++nnz;
                    }
                }
    }
    finish_agent(A, s, xi, yi, zi, Fx, Fy, Fz, is_static, nnz, c);
}

template <bool kStats>
__device__ __forceinline__ void flush_counts(const Counts &c, DevScalars *sc, int fuse) {
    if (fuse) {  // exact min/max of the new positions -> the next grid build's a1
        double v[7] = {c.lo0, c.lo1, c.lo2, c.hi0, c.hi1, c.hi2, c.dmax};
#pragma unroll
        for (int q = 0; q < 7; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double t = __shfl_xor_sync(0xffffffffu, v[q], o);
                v[q] = q < 3 ? fmin(v[q], t) : fmax(v[q], t);
            }
        if ((threadIdx.x & 31) == 0) {
            for (int q = 0; q < 3; ++q) atomicMin(&sc->enc_lo[q], enc_double(v[q]));
            for (int q = 0; q < 3; ++q) atomicMax(&sc->enc_hi[q], enc_double(v[3 + q]));
            atomicMax(&sc->enc_dmax, enc_double(v[6]));
        }
    }
    if (!kStats) return;
    const unsigned long long a = warp_sum_u64(c.cand), b = warp_sum_u64(c.nbr),
                             d = warp_sum_u64(c.cont), e = warp_sum_u64(c.stat),
                             f = warp_sum_u64(c.moved);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sc->stats[0], a);
        atomicAdd(&sc->stats[1], b);
        atomicAdd(&sc->stats[2], d);
        atomicAdd(&sc->stats[3], e);
        atomicAdd(&sc->stats[4], f);
    }
}


// the row-broadcast tile kernel (kernels_row.cu)
bdm_status launch_mech_row(Ctx *c, const MechArgs &A, bool stats, cudaStream_t st);

}  // namespace bdm
