/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the BioDynaMo/TeraAgent
 * mechanics hot path (arXiv 2503.10796, L. Breitwieser, ETH Diss. 30705).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or execute anything under oracle/.
 * The product path (paper_2503_10796_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b (section / equation label
 * given alongside).  Readings of passages where the paper is silent are numbered
 * R1..Rn and listed in DESIGN.md section 3 ("Readings").
 *
 * Arithmetic: IEEE binary64, round-to-nearest-even, compiled with
 * -O2 -ffp-contract=off so that the compiler never fuses a*b+c.  fma() is called at
 * exactly the two canonical sites (squared distance, force accumulation; R9).
 * sqrt() and '/' are IEEE correctly-rounded.
 *
 * Everything here is written for readability, not speed: sorting by qsort, box
 * lookup by binary search, one agent at a time.
 */
#define _USE_MATH_DEFINES
#include <math.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------ */
/* Counter-based PRNG: Philox4x32-10 (Salmon et al., SC'11 "Random123").            */
/* The paper proposes a per-agent counter-based PRNG as its remedy for              */
/* non-determinism: "Counter-based PRNGs [random123] could be a good choice"        */
/* (sec. "Reproducibility").  Reading R22: key = seed (lo, hi),        */
/* counter = (id_lo, id_hi, word2, stream).                                         */
/* ------------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {              /* key schedule: bump by the Weyl constants */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox words -> reals (reading R29).  Both conversions are exact in binary64. */
double orc_u32(uint32_t w) { return (double)w * 0x1p-32; }

double orc_u53(uint32_t wa, uint32_t wb)
{
    double hi = (double)(wa >> 5);   /* 27 bits */
    double lo = (double)(wb >> 6);   /* 26 bits */
    return (hi * 67108864.0 + lo) * 0x1p-53;
}

static void philox_draw(uint64_t seed, uint64_t id, uint32_t word2, uint32_t stream, uint32_t w[4])
{
    uint32_t ctr[4] = {(uint32_t)id, (uint32_t)(id >> 32), word2, stream};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, w);
}

/* ------------------------------------------------------------------------------ */
/* Agent flag bits (reading R8/R31).                                                */
/* ------------------------------------------------------------------------------ */
enum {
    ORC_MOVED = 1u << 0,   /* displacement != 0 in the last step                       */
    ORC_GREW = 1u << 1,    /* diameter increased in the last step                      */
    ORC_ADDED = 1u << 2,   /* agent created in the last step (initial agents included) */
    ORC_STATIC = 1u << 3,  /* force skipped in the last step                           */
    ORC_NNZ_SHIFT = 4,     /* bits 4-5: #nonzero neighbour forces, saturating at 2     */
};

/* ------------------------------------------------------------------------------ */
/* Population generation (ModelInitializer): uniform in a cube.        */
/* x,y from ctr (id, 0xFFFFFFFF, 2); z from (id, 0xFFFFFFFE, 2); a random diameter  */
/* d = d_lo + d_width*u from (id, 0xFFFFFFFD, 2) (reading R23).                      */
/* All initial agents carry ORC_ADDED: they "were added" before step 0, so          */
/* condition (iii) of P:4941-4946 prevents anyone from being static at step 0.      */
/* ------------------------------------------------------------------------------ */
void orc_init_spheres(int64_t id0, int64_t n, uint64_t seed, double side,
                      double d_lo, double d_width, int d_random,
                      double *x, double *y, double *z, double *d,
                      uint32_t *id, uint32_t *flags)
{
    for (int64_t k = 0; k < n; ++k) {
        uint64_t a = (uint64_t)(id0 + k);
        uint32_t w[4];
        philox_draw(seed, a, 0xFFFFFFFFu, 2u, w);
        x[k] = orc_u53(w[0], w[1]) * side;
        y[k] = orc_u53(w[2], w[3]) * side;
        philox_draw(seed, a, 0xFFFFFFFEu, 2u, w);
        z[k] = orc_u53(w[0], w[1]) * side;
        if (d_random) {
            philox_draw(seed, a, 0xFFFFFFFDu, 2u, w);
            d[k] = d_lo + d_width * orc_u53(w[0], w[1]);
        } else {
            d[k] = d_lo;
        }
        id[k] = (uint32_t)a;
        flags[k] = ORC_ADDED;
    }
}

/* ------------------------------------------------------------------------------ */
/* Morton order (fig:load-balancing-design): interleave the bits of    */
/* the box coordinates, coordinate 0 (x) in the lowest bit.                          */
/* ------------------------------------------------------------------------------ */
uint64_t orc_morton(const uint32_t *coord, int ndim, int bits)
{
    uint64_t code = 0;
    for (int b = 0; b < bits; ++b)
        for (int a = 0; a < ndim; ++a)
            code |= (uint64_t)((coord[a] >> b) & 1u) << (b * ndim + a);
    return code;
}

/* Blocked Morton key (reading R32): boxes are grouped in 4x4x4 tiles; tiles are    */
/* numbered row-major (x fastest); inside a tile the 64 boxes follow 3-D Morton.    */
uint64_t orc_blocked_key(int64_t bx, int64_t by, int64_t bz, const int64_t D[3])
{
    int64_t Tx = (D[0] + 3) / 4, Ty = (D[1] + 3) / 4;
    int64_t tile = ((bz / 4) * Ty + (by / 4)) * Tx + (bx / 4);
    uint32_t c[3] = {(uint32_t)(bx % 4), (uint32_t)(by % 4), (uint32_t)(bz % 4)};
    return (uint64_t)tile * 64u + orc_morton(c, 3, 2);
}

/* ------------------------------------------------------------------------------ */
/* Uniform grid geometry ("Environment Search"; P:4487-4530 sec:grid).  */
/* R = largest diameter ("box size ... determined automatically based on the        */
/* largest agent") unless the caller fixes it; L = R(1+2^-20) (R5);    */
/* origin = per-axis minimum (open boundary: "space grows to encapsulate all        */
/* agents"; R12).                                                           */
/* ------------------------------------------------------------------------------ */
typedef struct {
    double R, L, o[3], hi[3];
    int64_t D[3];
    double side;   /* > 0: toroidal cube [0, side)^3 (boundary 2, reading R52) */
} orc_grid;

void orc_grid_geometry(int64_t n, const double *x, const double *y, const double *z,
                       const double *d, double radius, double *out_R, double *out_L,
                       double out_o[3], int64_t out_D[3])
{
    double R = 0.0, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
        double p[3] = {x[i], y[i], z[i]};
        for (int a = 0; a < 3; ++a) {
            if (i == 0 || p[a] < lo[a]) lo[a] = p[a];
            if (i == 0 || p[a] > hi[a]) hi[a] = p[a];
        }
        if (d[i] > R) R = d[i];
    }
    if (radius > 0.0) R = radius;
    double L = R * (1.0 + 0x1p-20);
    for (int a = 0; a < 3; ++a) {
        out_o[a] = lo[a];
        out_D[a] = n > 0 ? (int64_t)floor((hi[a] - lo[a]) / L) + 1 : 0;
    }
    *out_R = R;
    *out_L = L;
}

static void box_of(const orc_grid *g, double px, double py, double pz, int64_t b[3])
{
    b[0] = (int64_t)floor((px - g->o[0]) / g->L);
    b[1] = (int64_t)floor((py - g->o[1]) / g->L);
    b[2] = (int64_t)floor((pz - g->o[2]) / g->L);
    if (g->side > 0.0)  /* toroidal: the last box also takes x == side (R20), R52 */
        for (int a = 0; a < 3; ++a) b[a] = b[a] < 0 ? 0 : (b[a] > g->D[a] - 1 ? g->D[a] - 1 : b[a]);
}

/* Toroidal grid (boundary 2, reading R52): the periodic cube [0, side)^3 of the paper's
 * toroidal boundary ("agents that leave the space on one side, will enter on the
 * opposite side"), with the lattice of R19: D = floor(side / R) boxes of edge
 * L = side / D per axis (D >= 3, so the 27 neighbour boxes are distinct). */
static int torus_geometry(orc_grid *g, double R, double side)
{
    int64_t D = (int64_t)floor(side / R);
    if (!(R > 0.0) || D < 3) return -1;
    g->R = R;
    g->L = side / (double)D;
    g->side = side;
    for (int a = 0; a < 3; ++a) {
        g->o[a] = 0.0;
        g->D[a] = D;
    }
    return 0;
}

/* ---- the grid itself: agents sorted by (row-major box index, id) ---------------- */
typedef struct {
    int64_t box;   /* (bz*Dy + by)*Dx + bx */
    uint32_t id;
    int64_t idx;   /* agent index in the input arrays */
} orc_entry;

static int cmp_entry(const void *pa, const void *pb)
{
    const orc_entry *a = pa, *b = pb;
    if (a->box != b->box) return a->box < b->box ? -1 : 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return 0;
}

typedef struct {
    orc_grid g;
    int64_t n;
    orc_entry *e;  /* n entries sorted by (box, id) */
} orc_index;

static int64_t lin_box(const orc_grid *g, int64_t bx, int64_t by, int64_t bz)
{
    return (bz * g->D[1] + by) * g->D[0] + bx;
}

/* frame (nullable): a global grid frame (o[3], R) shared by the ranks of a
 * partitioned run: the origin and R come from it, the box count from the
 * agents' extent measured from that origin. */
static void index_build(orc_index *ix, int64_t n, const double *x, const double *y,
                        const double *z, const double *d, const uint32_t *id, double radius,
                        const double *frame, double torus_side)
{
    ix->n = n;
    orc_grid_geometry(n, x, y, z, d, radius, &ix->g.R, &ix->g.L, ix->g.o, ix->g.D);
    ix->g.side = 0.0;
    if (torus_side > 0.0) torus_geometry(&ix->g, ix->g.R, torus_side);
    if (frame) {
        double R = radius > 0.0 ? radius : frame[3];
        double L = R * (1.0 + 0x1p-20);
        ix->g.R = R;
        ix->g.L = L;
        for (int a = 0; a < 3; ++a) {
            double hi = frame[a];
            const double *p = a == 0 ? x : a == 1 ? y : z;
            for (int64_t i = 0; i < n; ++i)
                if (p[i] > hi) hi = p[i];
            ix->g.o[a] = frame[a];
            ix->g.D[a] = (int64_t)floor((hi - frame[a]) / L) + 1;
        }
    }
    ix->e = (orc_entry *)malloc(sizeof(orc_entry) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        int64_t b[3];
        box_of(&ix->g, x[i], y[i], z[i], b);
        ix->e[i].box = lin_box(&ix->g, b[0], b[1], b[2]);
        ix->e[i].id = id[i];
        ix->e[i].idx = i;
    }
    qsort(ix->e, (size_t)n, sizeof(orc_entry), cmp_entry);
}

static void index_free(orc_index *ix) { free(ix->e); }

/* [first, last) range of entries in box `box` (binary search) */
static void box_range(const orc_index *ix, int64_t box, int64_t *first, int64_t *last)
{
    int64_t lo = 0, hi = ix->n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (ix->e[mid].box < box) lo = mid + 1; else hi = mid;
    }
    *first = lo;
    hi = ix->n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (ix->e[mid].box <= box) lo = mid + 1; else hi = mid;
    }
    *last = lo;
}

/* Squared centre distance in the canonical operation order (R9):
 * D = fma(dz, dz, fma(dy, dy, dx*dx)) with d* = (own - other). */
static double sqdist(double dx, double dy, double dz)
{
    return fma(dz, dz, fma(dy, dy, dx * dx));
}

/* ------------------------------------------------------------------------------ */
/* Neighbour pairs by the plain definition (all pairs; reading R4):                 */
/* N_i = { j != i : D_ij <= R*R }.  Writes (id_i << 32 | id_j) for every ordered     */
/* pair, unsorted; returns the count (pairs beyond `cap` are counted, not written). */
/* ------------------------------------------------------------------------------ */
int64_t orc_neighbor_pairs_brute(int64_t n, const double *x, const double *y, const double *z,
                                 const uint32_t *id, double R, uint64_t *pairs, int64_t cap)
{
    double R2 = R * R;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double D = sqdist(x[i] - x[j], y[i] - y[j], z[i] - z[j]);
            if (D <= R2) {
                if (cnt < cap) pairs[cnt] = ((uint64_t)id[i] << 32) | id[j];
                ++cnt;
            }
        }
    return cnt;
}

/* Same relation enumerated through the uniform grid's 27 boxes. */
int64_t orc_neighbor_pairs_grid(int64_t n, const double *x, const double *y, const double *z,
                                const double *d, const uint32_t *id, double radius,
                                uint64_t *pairs, int64_t cap)
{
    orc_index ix;
    index_build(&ix, n, x, y, z, d, id, radius, NULL, 0.0);
    double R2 = ix.g.R * ix.g.R;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t b[3];
        box_of(&ix.g, x[i], y[i], z[i], b);
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t cx = b[0] + dx, cy = b[1] + dy, cz = b[2] + dz;
                    if (cx < 0 || cy < 0 || cz < 0 || cx >= ix.g.D[0] || cy >= ix.g.D[1] ||
                        cz >= ix.g.D[2])
                        continue;
                    int64_t f, l;
                    box_range(&ix, lin_box(&ix.g, cx, cy, cz), &f, &l);
                    for (int64_t s = f; s < l; ++s) {
                        int64_t j = ix.e[s].idx;
                        if (j == i) continue;
                        double D = sqdist(x[i] - x[j], y[i] - y[j], z[i] - z[j]);
                        if (D <= R2) {
                            if (cnt < cap) pairs[cnt] = ((uint64_t)id[i] << 32) | id[j];
                            ++cnt;
                        }
                    }
                }
    }
    index_free(&ix);
    return cnt;
}

/* ------------------------------------------------------------------------------ */
/* Pair force, Eq. 4.1 / 4.2 (eq:force, eq:force-radius):               */
/*   F_N = k*delta - gamma*sqrt(rbar*delta),  rbar = r1*r2/(r1+r2)                   */
/* delta = r_i + r_j - |x_i - x_j| (R2), force only for delta > 0 (R3) and          */
/* dist > 0 (R10).  Direction along the centre line, positive = repulsive (R1).     */
/* Returns F_N, writes s = F_N / dist.                                               */
/* ------------------------------------------------------------------------------ */
double orc_pair_force(double k, double gamma, double D, double ri, double rj, int *contact,
                      double *s_out)
{
    double dist = sqrt(D);
    double delta = (ri + rj) - dist;
    *contact = 0;
    *s_out = 0.0;
    if (!(delta > 0.0 && dist > 0.0)) return 0.0;
    *contact = 1;
    double rbar = (ri * rj) / (ri + rj);
    double Fn = k * delta - gamma * sqrt(rbar * delta);
    *s_out = Fn / dist;
    return Fn;
}

/* ------------------------------------------------------------------------------ */
/* One mechanics step (MechanicalForcesOp + BoundSpaceOp,  */
/* with the static-agent skip of sec:static-agents).  Copy (Jacobi)     */
/* semantics: every read uses the start-of-step state (R11).            */
/* ------------------------------------------------------------------------------ */
typedef struct {
    double k, gamma, dt, max_disp, force_threshold, radius;
    int32_t detect_static, boundary;  /* boundary: 0 open, 1 closed */
    double lo[3], hi[3];
    int32_t use_frame, pad_;          /* 1: grid frame below instead of the agents' own */
    double frame[4];                  /* o[3], R (global frame)            */
} orc_mech_params;

typedef struct {
    int64_t cand, nbr, cont, n_static;
} orc_counters;

static int nnz_of(uint32_t f) { return (int)((f >> ORC_NNZ_SHIFT) & 3u); }

double orc_wrap(double el, double max_bound);

/* Toroidal difference (R52): the minimum image of own - other per axis, as Alg. 7's
 * periodic search (R19): d > side/2 -> d - side, d < -side/2 -> d + side. */
static double torus_diff(const orc_grid *g, double v)
{
    if (!(g->side > 0.0)) return v;
    double half = g->side * 0.5;
    if (v > half) return v - g->side;
    if (v < -half) return v + g->side;
    return v;
}

/* Neighbour box c + off along one axis: -1 if outside an open/closed grid; wrapped
 * periodically on the torus. */
static int64_t nbr_box(const orc_grid *g, int64_t c, int a)
{
    if (g->side > 0.0) return c < 0 ? c + g->D[a] : (c >= g->D[a] ? c - g->D[a] : c);
    return (c < 0 || c >= g->D[a]) ? -1 : c;
}

/* Computes the step for agents idx_list[0..m) (all agents when idx_list == NULL;
 * then m must equal n).  Results are written at position k of the out arrays for
 * the k-th listed agent. */
void orc_mech_step(int64_t n, const double *x, const double *y, const double *z,
                   const double *d, const uint32_t *id, const uint32_t *flags,
                   const orc_mech_params *p, int64_t m, const int64_t *idx_list,
                   double *x_out, double *y_out, double *z_out, uint32_t *flags_out,
                   double *force_out /* nullable: 3*m, the summed force F_i */,
                   orc_counters *cnt)
{
    memset(cnt, 0, sizeof(*cnt));
    if (n == 0) return;
    double torus = 0.0;
    if (p->boundary == 2) {  /* R52: the cube [0, hi[0])^3, at least 3 boxes per axis */
        torus = p->hi[0];
        orc_grid chk;
        double R = p->radius;
        if (!(R > 0.0))
            for (int64_t i = 0; i < n; ++i) R = d[i] > R ? d[i] : R;
        if (p->lo[0] != 0.0 || p->lo[1] != 0.0 || p->lo[2] != 0.0 || p->hi[1] != torus ||
            p->hi[2] != torus || torus_geometry(&chk, R, torus) != 0) {
            cnt->n_static = -1;  /* invalid torus: nothing computed */
            return;
        }
    }
    orc_index ix;
    index_build(&ix, n, x, y, z, d, id, p->radius, p->use_frame ? p->frame : NULL, torus);
    const orc_grid *g = &ix.g;
    double R2 = g->R * g->R;
    const uint32_t CHANGED = ORC_MOVED | ORC_GREW | ORC_ADDED;

    for (int64_t k = 0; k < m; ++k) {
        int64_t i = idx_list ? idx_list[k] : k;
        int64_t b[3];
        box_of(g, x[i], y[i], z[i], b);
        double ri = d[i] * 0.5;

        /* (a5) static classification: (i) the agent and none of its
         * neighbours moved, (ii) no force-increasing change (growth), (iii) no agent
         * added within the radius, (iv) at most one non-zero neighbour force.  All
         * facts refer to the last iteration (flags of step t-1); the neighbours are
         * those within R now (R8). */
        int is_static = 0;
        if (p->detect_static && !(flags[i] & CHANGED) && nnz_of(flags[i]) <= 1) {
            is_static = 1;
            for (int dz = -1; dz <= 1 && is_static; ++dz)
                for (int dy = -1; dy <= 1 && is_static; ++dy)
                    for (int dx = -1; dx <= 1 && is_static; ++dx) {
                        int64_t cx = nbr_box(g, b[0] + dx, 0), cy = nbr_box(g, b[1] + dy, 1),
                                cz = nbr_box(g, b[2] + dz, 2);
                        if (cx < 0 || cy < 0 || cz < 0) continue;
                        int64_t f, l;
                        box_range(&ix, lin_box(g, cx, cy, cz), &f, &l);
                        for (int64_t s = f; s < l; ++s) {
                            int64_t j = ix.e[s].idx;
                            if (j == i) continue;
                            double D = sqdist(torus_diff(g, x[i] - x[j]), torus_diff(g, y[i] - y[j]),
                                              torus_diff(g, z[i] - z[j]));
                            if (D <= R2 && (flags[j] & CHANGED)) {
                                is_static = 0;
                                break;
                            }
                        }
                    }
        }

        double Dx = 0.0, Dy = 0.0, Dz = 0.0;
        double Fx = 0.0, Fy = 0.0, Fz = 0.0;
        int nnz;
        if (is_static) {
            nnz = nnz_of(flags[i]);  /* carried */
            cnt->n_static++;
        } else {
            /* (a6)+(a7): 27 boxes in (dz, dy, dx) lexicographic order, inside a box
             * ascending id (R9); sum f_ij = s*(x_i - x_j) with fma. */
            nnz = 0;
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        int64_t cx = nbr_box(g, b[0] + dx, 0), cy = nbr_box(g, b[1] + dy, 1),
                                cz = nbr_box(g, b[2] + dz, 2);
                        if (cx < 0 || cy < 0 || cz < 0) continue;
                        int64_t f, l;
                        box_range(&ix, lin_box(g, cx, cy, cz), &f, &l);
                        for (int64_t s = f; s < l; ++s) {
                            int64_t j = ix.e[s].idx;
                            if (j == i) continue;
                            cnt->cand++;
                            double ex = torus_diff(g, x[i] - x[j]), ey = torus_diff(g, y[i] - y[j]),
                                   ez = torus_diff(g, z[i] - z[j]);
                            double D = sqdist(ex, ey, ez);
                            if (!(D <= R2)) continue;
                            cnt->nbr++;
                            int contact;
                            double sc;
                            double Fn = orc_pair_force(p->k, p->gamma, D, ri, d[j] * 0.5,
                                                       &contact, &sc);
                            if (!contact) continue;
                            cnt->cont++;
                            Fx = fma(sc, ex, Fx);
                            Fy = fma(sc, ey, Fy);
                            Fz = fma(sc, ez, Fz);
                            if (Fn != 0.0 && nnz < 2) ++nnz;
                        }
                    }
            /* (a8) displacement = dt * F (R6); no move unless |F| > threshold (R7,
             * P:4964-4965); cap |displacement| at max_disp. */
            double F2 = Fx * Fx + Fy * Fy + Fz * Fz;
            double tau = p->force_threshold;
            if (F2 > tau * tau) {
                Dx = p->dt * Fx;
                Dy = p->dt * Fy;
                Dz = p->dt * Fz;
                double n2 = Dx * Dx + Dy * Dy + Dz * Dz;
                double mx = p->max_disp;
                if (n2 > mx * mx) {
                    double scale = mx / sqrt(n2);
                    Dx = Dx * scale;
                    Dy = Dy * scale;
                    Dz = Dz * scale;
                }
            }
        }
        double nx = x[i] + Dx, ny = y[i] + Dy, nz = z[i] + Dz;
        /* (a9) boundary condition (sec:space-boundary): open = no-op (the
         * grid origin follows the agents, R12); closed = clamp into [lo, hi]. */
        if (p->boundary == 1) {
            double *q[3] = {&nx, &ny, &nz};
            for (int a = 0; a < 3; ++a) {
                if (*q[a] < p->lo[a]) *q[a] = p->lo[a];
                if (*q[a] > p->hi[a]) *q[a] = p->hi[a];
            }
        } else if (p->boundary == 2) {  /* toroidal: Alg. 9's literal wrap (R20, R52) */
            nx = orc_wrap(nx, torus);
            ny = orc_wrap(ny, torus);
            nz = orc_wrap(nz, torus);
        }
        int moved = (Dx != 0.0 || Dy != 0.0 || Dz != 0.0);
        if (force_out) {
            force_out[3 * k + 0] = Fx;
            force_out[3 * k + 1] = Fy;
            force_out[3 * k + 2] = Fz;
        }
        x_out[k] = nx;
        y_out[k] = ny;
        z_out[k] = nz;
        flags_out[k] = (moved ? ORC_MOVED : 0u) | (is_static ? ORC_STATIC : 0u) |
                       ((uint32_t)nnz << ORC_NNZ_SHIFT);
    }
    index_free(&ix);
}

/* ------------------------------------------------------------------------------ */
/* The agent order after a step (A12): agents sorted by the blocked     */
/* Morton key of their box in the step's grid, ascending id inside a box.            */
/* Writes the permutation (input indices in sorted order) and the keys.              */
/* ------------------------------------------------------------------------------ */
typedef struct {
    uint64_t key;
    uint32_t id;
    int64_t idx;
} orc_kentry;

static int cmp_kentry(const void *pa, const void *pb)
{
    const orc_kentry *a = pa, *b = pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return 0;
}

/* torus_side > 0: the toroidal lattice of R52 (boxes clamped to D - 1, R20) */
void orc_sorted_order_torus(int64_t n, const double *x, const double *y, const double *z,
                            const double *d, const uint32_t *id, double radius, double torus_side,
                            int64_t *perm, uint64_t *keys_sorted)
{
    if (n == 0) return;
    orc_grid g;
    orc_grid_geometry(n, x, y, z, d, radius, &g.R, &g.L, g.o, g.D);
    g.side = 0.0;
    if (torus_side > 0.0 && torus_geometry(&g, g.R, torus_side) != 0) return;
    orc_kentry *e = (orc_kentry *)malloc(sizeof(orc_kentry) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t b[3];
        box_of(&g, x[i], y[i], z[i], b);
        e[i].key = orc_blocked_key(b[0], b[1], b[2], g.D);
        e[i].id = id[i];
        e[i].idx = i;
    }
    qsort(e, (size_t)n, sizeof(orc_kentry), cmp_kentry);
    for (int64_t i = 0; i < n; ++i) {
        perm[i] = e[i].idx;
        if (keys_sorted) keys_sorted[i] = e[i].key;
    }
    free(e);
}

void orc_sorted_order(int64_t n, const double *x, const double *y, const double *z,
                      const double *d, const uint32_t *id, double radius, int64_t *perm,
                      uint64_t *keys_sorted)
{
    orc_sorted_order_torus(n, x, y, z, d, id, radius, 0.0, perm, keys_sorted);
}

/* ------------------------------------------------------------------------------ */
/* Growth and division (cfg3): Alg. 4 control flow "grow if d < max, else divide"   */
/* (algo:tumor_growth_module) with division probability 1; Cell::Divide */
/* splits the volume by the volume ratio and places the daughter along the division */
/* axis; additions become visible at the next iteration (*/
/* P:4538-4544).  Readings R13-R15, R28.                                 */
/* ------------------------------------------------------------------------------ */

/* R28: deterministic cube root.  v = m 2^e (frexp, m in [0.5,1)); start y = 2^k with
 * k = floor((e+1)/3); exactly 8 Newton steps y <- (2y + v/(y*y))/3, no fma. */
double orc_cbrt_det(double v)
{
    if (!(v > 0.0)) return 0.0;
    int e;
    (void)frexp(v, &e);
    int num = e + 1;
    int k = num >= 0 ? num / 3 : -((-num + 2) / 3); /* mathematical floor(num/3) */
    double y = ldexp(1.0, k);
    for (int it = 0; it < 8; ++it) {
        double yy = y * y;
        double q = v / yy;
        double t = 2.0 * y + q;
        y = t / 3.0;
    }
    return y;
}

/* R13: division axis uniform on the sphere by rejection in the unit ball.  Try k uses
 * Philox counter (id, step, 3 + 4k): v_a = 2 u32(w_a) - 1 (a = 0,1,2); accept if
 * 0 < v.v <= 1, u = v / sqrt(v.v); after 16 rejected tries the axis is +x. */
void orc_division_axis(uint64_t seed, uint64_t id, uint32_t step, double u[3])
{
    for (uint32_t k = 0; k < 16; ++k) {
        uint32_t w[4];
        philox_draw(seed, id, step, 3u + 4u * k, w);
        double vx = 2.0 * orc_u32(w[0]) - 1.0;
        double vy = 2.0 * orc_u32(w[1]) - 1.0;
        double vz = 2.0 * orc_u32(w[2]) - 1.0;
        double n2 = vx * vx + vy * vy + vz * vz;
        if (n2 > 0.0 && n2 <= 1.0) {
            double n = sqrt(n2);
            u[0] = vx / n;
            u[1] = vy / n;
            u[2] = vz / n;
            return;
        }
    }
    u[0] = 1.0;
    u[1] = 0.0;
    u[2] = 0.0;
}

/* One growth/division pass over n agents that already carry their post-mechanics
 * positions (R15: growth and division read the start-of-step volume V).  For every
 * agent in ascending id order:
 *   V < v_max:  V += growth; d = 2 cbrt_det(V C), C = 0.75/M_PI; flag GREW if d grew
 *   else:       V <- V/2 for mother and daughter (volume ratio 0.5, exact),
 *               r' = cbrt_det(V' C), d' = 2r', axis u (R13),
 *               mother at x - r'u (flag MOVED, its diameter shrank),
 *               daughter at x + r'u (flag ADDED), id = n + rank among dividers by id,
 *               appended at index n + rank.
 * Arrays must have room for the daughters; returns the new agent count.
 * Input arrays may be in any order; ids must be exactly 0..n-1. */
int64_t orc_grow_divide(int64_t n, double *x, double *y, double *z, double *d, double *vol,
                        uint32_t *id, uint32_t *flags, int64_t capacity, double growth,
                        double v_max, uint64_t seed, uint32_t step)
{
    const double C = 0.75 / M_PI;
    int64_t *by_id = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) by_id[id[i]] = i;
    int64_t ndiv = 0;
    for (int64_t k = 0; k < n; ++k)
        if (!(vol[by_id[k]] < v_max)) ++ndiv;
    if (n + ndiv > capacity) {
        free(by_id);
        return -(n + ndiv);
    }
    int64_t rank = 0;
    for (int64_t k = 0; k < n; ++k) {      /* ascending id */
        int64_t i = by_id[k];
        double V = vol[i];
        if (V < v_max) {
            double Vn = V + growth;
            double dn = 2.0 * orc_cbrt_det(Vn * C);
            if (dn > d[i]) flags[i] |= ORC_GREW;
            vol[i] = Vn;
            d[i] = dn;
        } else {
            double Vh = V * 0.5;
            double r = orc_cbrt_det(Vh * C);
            double u[3];
            orc_division_axis(seed, id[i], step, u);
            int64_t j = n + rank;
            double px = x[i], py = y[i], pz = z[i];
            x[i] = px - r * u[0];
            y[i] = py - r * u[1];
            z[i] = pz - r * u[2];
            x[j] = px + r * u[0];
            y[j] = py + r * u[1];
            z[j] = pz + r * u[2];
            vol[i] = Vh;
            vol[j] = Vh;
            d[i] = 2.0 * r;
            d[j] = 2.0 * r;
            flags[i] |= ORC_MOVED;
            flags[j] = ORC_ADDED;
            id[j] = (uint32_t)(n + rank);
            ++rank;
        }
    }
    free(by_id);
    return n + ndiv;
}

/* ------------------------------------------------------------------------------ */
/* SIR epidemiology step (cfg4): Algorithms 7-9 (algo:infection P:3220-3249,        */
/* algo:recovery P:3251-3270, algo:random-movement P:3272-3303).  Readings:          */
/*   R16  movement v = 2u - 1 per axis, capped: if v.v > 1 then v = v / sqrt(v.v)   */
/*   R17  draws compared with '<' (u = w 2^-32)                                      */
/*   R18  order infection -> recovery -> movement; neighbours' states and positions  */
/*        from the start-of-step snapshot; own state updated in sequence             */
/*   R19  periodic neighbour search with minimum-image differences                    */
/*   R20  Alg. 9 wrap taken literally: el = fmod(el, max); if el < 0: el = max + el   */
/*   R22  Philox counter (id, step, 0) -> movement w0..w2 + infection w3;             */
/*        (id, step, 1) -> recovery w0                                              */
/* No fused multiply-add anywhere (BASELINE: "FMA contraction off").                 */
/* ------------------------------------------------------------------------------ */
enum { ORC_S = 0, ORC_I = 1, ORC_R = 2 };

double orc_wrap(double el, double max_bound)
{
    el = fmod(el, max_bound);
    if (el < 0.0) el = max_bound + el;
    return el;
}

static double min_image(double d, double side)
{
    double half = side * 0.5;
    if (d > half) d = d - side;
    else if (d < -half) d = d + side;
    return d;
}

typedef struct {
    int64_t key;   /* (bz*D + by)*D + bx */
    int64_t idx;
} orc_kv;

static int cmp_kv(const void *pa, const void *pb)
{
    const orc_kv *a = pa, *b = pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

static int64_t sir_box(double v, double L, int64_t D)
{
    int64_t b = (int64_t)floor(v / L);
    if (b < 0) b = 0;
    if (b > D - 1) b = D - 1;
    return b;
}

/* Updates x, y, z, state in place for n agents in a periodic cube [0, side)^3 with
 * D = floor(side / radius) boxes of edge L = side / D per axis (needs D >= 3).
 * counts[0..2] receives S, I, R after the step; returns the number of new infections. */
/* Sampled form: computes the step for the m agents idx[0..m) (NULL: all, m = n) from
 * the full snapshot (x, y, z, state) and writes their new values to the out arrays
 * (position k for the k-th listed agent).  Inputs are not modified. */
int64_t orc_sir_step_sample(int64_t n, const double *x, const double *y, const double *z,
                            const uint8_t *state, const uint32_t *id, double side,
                            double radius, double p_inf, double p_rec, uint64_t seed,
                            uint32_t step, int64_t m, const int64_t *idx, double *ox,
                            double *oy, double *oz, uint8_t *ostate, int64_t counts[3]);

int64_t orc_sir_step(int64_t n, double *x, double *y, double *z, uint8_t *state,
                     const uint32_t *id, double side, double radius, double p_inf,
                     double p_rec, uint64_t seed, uint32_t step, int64_t counts[3])
{
    double *ox = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *oy = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *oz = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    uint8_t *os = malloc((size_t)(n > 0 ? n : 1));
    int64_t r = orc_sir_step_sample(n, x, y, z, state, id, side, radius, p_inf, p_rec, seed,
                                    step, n, NULL, ox, oy, oz, os, counts);
    memcpy(x, ox, sizeof(double) * (size_t)n);
    memcpy(y, oy, sizeof(double) * (size_t)n);
    memcpy(z, oz, sizeof(double) * (size_t)n);
    memcpy(state, os, (size_t)n);
    free(ox); free(oy); free(oz); free(os);
    return r;
}

int64_t orc_sir_step_sample(int64_t n, const double *x, const double *y, const double *z,
                            const uint8_t *state, const uint32_t *id, double side,
                            double radius, double p_inf, double p_rec, uint64_t seed,
                            uint32_t step, int64_t m, const int64_t *idx, double *ox,
                            double *oy, double *oz, uint8_t *ostate, int64_t counts[3])
{
    int64_t D = (int64_t)floor(side / radius);
    double L = side / (double)D;
    double R2 = radius * radius;
    const double *x0 = x, *y0 = y, *z0 = z;   /* the snapshot (inputs are read-only) */
    const uint8_t *s0 = state;
    /* index of the infected agents of the snapshot, sorted by box */
    int64_t ni = 0;
    for (int64_t i = 0; i < n; ++i) ni += (s0[i] == ORC_I);
    orc_kv *inf = malloc(sizeof(orc_kv) * (size_t)(ni > 0 ? ni : 1));
    ni = 0;
    for (int64_t i = 0; i < n; ++i)
        if (s0[i] == ORC_I) {
            int64_t bx = sir_box(x0[i], L, D), by = sir_box(y0[i], L, D), bz = sir_box(z0[i], L, D);
            inf[ni].key = (bz * D + by) * D + bx;
            inf[ni].idx = i;
            ++ni;
        }
    qsort(inf, (size_t)ni, sizeof(orc_kv), cmp_kv);

    int64_t new_inf = 0;
    counts[0] = counts[1] = counts[2] = 0;
    for (int64_t k = 0; k < m; ++k) {
        int64_t i = idx ? idx[k] : k;
        uint32_t w[4];
        philox_draw(seed, id[i], step, 0u, w);
        uint8_t st = s0[i];
        /* Alg. 7: a susceptible agent, with probability p_inf, becomes infected if an
         * infected agent is within the infection radius */
        if (st == ORC_S && orc_u32(w[3]) < p_inf) {
            int64_t bx = sir_box(x0[i], L, D), by = sir_box(y0[i], L, D), bz = sir_box(z0[i], L, D);
            int found = 0;
            for (int dz = -1; dz <= 1 && !found; ++dz)
                for (int dy = -1; dy <= 1 && !found; ++dy)
                    for (int dx = -1; dx <= 1 && !found; ++dx) {
                        int64_t cx = ((bx + dx) % D + D) % D, cy = ((by + dy) % D + D) % D,
                                cz = ((bz + dz) % D + D) % D;
                        int64_t key = (cz * D + cy) * D + cx;
                        int64_t lo = 0, hi = ni;
                        while (lo < hi) {
                            int64_t mid = (lo + hi) / 2;
                            if (inf[mid].key < key) lo = mid + 1; else hi = mid;
                        }
                        for (int64_t s = lo; s < ni && inf[s].key == key; ++s) {
                            int64_t j = inf[s].idx;
                            double ex = min_image(x0[i] - x0[j], side);
                            double ey = min_image(y0[i] - y0[j], side);
                            double ez = min_image(z0[i] - z0[j], side);
                            double Dd = ex * ex + ey * ey + ez * ez;
                            if (Dd <= R2) { found = 1; break; }
                        }
                    }
            if (found) {
                st = ORC_I;
                ++new_inf;
            }
        }
        /* Alg. 8: an infected agent recovers with probability p_rec */
        if (st == ORC_I) {
            uint32_t wr[4];
            philox_draw(seed, id[i], step, 1u, wr);
            if (orc_u32(wr[0]) < p_rec) st = ORC_R;
        }
        ostate[k] = st;
        counts[st] += 1;
        /* Alg. 9: random movement, capped at unit length (R16), toroidal wrap (R20) */
        double vx = 2.0 * orc_u32(w[0]) - 1.0;
        double vy = 2.0 * orc_u32(w[1]) - 1.0;
        double vz = 2.0 * orc_u32(w[2]) - 1.0;
        double v2 = vx * vx + vy * vy + vz * vz;
        if (v2 > 1.0) {
            double nv = sqrt(v2);
            vx = vx / nv;
            vy = vy / nv;
            vz = vz / nv;
        }
        ox[k] = orc_wrap(x0[i] + vx, side);
        oy[k] = orc_wrap(y0[i] + vy, side);
        oz[k] = orc_wrap(z0[i] + vz, side);
    }
    free(inf);
    return new_inf;
}

/* Population for cfg4: uniform in [0, side)^3 (same per-id recipe as the spheres),
 * ids < n_infected start infected (R21), all others susceptible. */
void orc_init_sir(int64_t n, uint64_t seed, double side, int64_t n_infected, double *x,
                  double *y, double *z, uint8_t *state, uint32_t *id)
{
    for (int64_t k = 0; k < n; ++k) {
        uint32_t w[4];
        philox_draw(seed, (uint64_t)k, 0xFFFFFFFFu, 2u, w);
        x[k] = orc_u53(w[0], w[1]) * side;
        y[k] = orc_u53(w[2], w[3]) * side;
        philox_draw(seed, (uint64_t)k, 0xFFFFFFFEu, 2u, w);
        z[k] = orc_u53(w[0], w[1]) * side;
        id[k] = (uint32_t)k;
        state[k] = (k < n_infected) ? ORC_I : ORC_S;
    }
}

/* ------------------------------------------------------------------------------ */
/* Extracellular diffusion, secretion and chemotaxis.         */
/* Grid (reading R34): nx*ny*nz points, point (i,j,k) stored at i + nx*(j + ny*k); */
/* point (i,j,k) is the centre of the cell [lo + i*dx, lo + (i+1)*dx) x ... and    */
/* values outside the grid are 0: "substances diffuse out of the simulation        */
/* space".                                                           */
/* ------------------------------------------------------------------------------ */
static double grid_at(const double *u, int64_t nx, int64_t ny, int64_t nz, int64_t i, int64_t j,
                      int64_t k)
{
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return 0.0;
    return u[i + nx * (j + ny * k)];
}

/* Eq. 4.3 (eq:centraldiff), one explicit step from u to out (distinct
 * arrays).  Reading R35 fixes the operation order: the decay factor 1 - mu*dt and the
 * coefficients nu*dt / (dx*dx) are computed once; per point
 *   v = u*(1 - mu dt);  v = v + cx*((u_{i+1} - 2u) + u_{i-1});  then the y and z terms,
 * each second difference left to right, no fused multiply-add. */
void orc_diffuse_step(int64_t nx, int64_t ny, int64_t nz, const double *u, double *out, double nu,
                      double mu, double dt, double dx, double dy, double dz)
{
    const double decay = 1.0 - mu * dt;
    const double cx = (nu * dt) / (dx * dx);
    const double cy = (nu * dt) / (dy * dy);
    const double cz = (nu * dt) / (dz * dz);
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const double c = u[i + nx * (j + ny * k)];
                double v = c * decay;
                v = v + cx * ((grid_at(u, nx, ny, nz, i + 1, j, k) - 2.0 * c) +
                              grid_at(u, nx, ny, nz, i - 1, j, k));
                v = v + cy * ((grid_at(u, nx, ny, nz, i, j + 1, k) - 2.0 * c) +
                              grid_at(u, nx, ny, nz, i, j - 1, k));
                v = v + cz * ((grid_at(u, nx, ny, nz, i, j, k + 1) - 2.0 * c) +
                              grid_at(u, nx, ny, nz, i, j, k - 1));
                out[i + nx * (j + ny * k)] = v;
            }
}

/* The cell containing a position (reading R36): floor((p - lo)/d), clamped to the grid. */
static int64_t grid_cell(double p, double lo, double d, int64_t n)
{
    double b = floor((p - lo) / d);
    if (b < 0.0) b = 0.0;
    if (b > (double)(n - 1)) b = (double)(n - 1);
    return (int64_t)b;
}

/* Alg. secretion_module: every agent of the selected type adds q to the
 * cell containing its position, agents in index order (R36).  For a constant q the
 * result does not depend on the order (every partial sum adds the same q). */
void orc_secrete(int64_t n, const double *x, const double *y, const double *z, const uint8_t *type,
                 int type_sel, double q, double *u, int64_t nx, int64_t ny, int64_t nz,
                 const double lo[3], double dx, double dy, double dz)
{
    for (int64_t a = 0; a < n; ++a) {
        if ((int)type[a] != type_sel) continue;
        const int64_t i = grid_cell(x[a], lo[0], dx, nx), j = grid_cell(y[a], lo[1], dy, ny),
                      k = grid_cell(z[a], lo[2], dz, nz);
        u[i + nx * (j + ny * k)] = u[i + nx * (j + ny * k)] + q;
    }
}

/* Alg. chemotaxis_module: agents of the selected type move by
 * weight * GetNormalizedGradient(pos).  Reading R37: the gradient is the central
 * difference at the cell of pos, g_a = (u_{+1} - u_{-1}) / (2 d_a) (outside = 0),
 * normalized as g / sqrt((gx*gx + gy*gy) + gz*gz) (zero gradient -> no move); R38:
 * p_a = p_a + weight * g_a. */
void orc_chemotaxis(int64_t n, double *x, double *y, double *z, const uint8_t *type, int type_sel,
                    double weight, const double *u, int64_t nx, int64_t ny, int64_t nz,
                    const double lo[3], double dx, double dy, double dz)
{
    for (int64_t a = 0; a < n; ++a) {
        if ((int)type[a] != type_sel) continue;
        const int64_t i = grid_cell(x[a], lo[0], dx, nx), j = grid_cell(y[a], lo[1], dy, ny),
                      k = grid_cell(z[a], lo[2], dz, nz);
        const double gx = (grid_at(u, nx, ny, nz, i + 1, j, k) - grid_at(u, nx, ny, nz, i - 1, j, k)) /
                          (2.0 * dx);
        const double gy = (grid_at(u, nx, ny, nz, i, j + 1, k) - grid_at(u, nx, ny, nz, i, j - 1, k)) /
                          (2.0 * dy);
        const double gz = (grid_at(u, nx, ny, nz, i, j, k + 1) - grid_at(u, nx, ny, nz, i, j, k - 1)) /
                          (2.0 * dz);
        const double n2 = gx * gx + gy * gy + gz * gz;
        if (!(n2 > 0.0)) continue;
        const double nrm = sqrt(n2);
        x[a] = x[a] + weight * (gx / nrm);
        y[a] = y[a] + weight * (gy / nrm);
        z[a] = z[a] + weight * (gz / nrm);
    }
}

/* ------------------------------------------------------------------------------ */
/* Oncology behaviour + agent removal.                          */
/* Alg. 4 (algo:tumor_growth_module) with the Table 4.2 parameters     */
/* and the parallel removal of sec. "Agent addition and removal"     */
/* (P:4545-4603).  Readings:                                             */
/*   R41  brownian = v / |v| with v = 2 u32(w0..w2) - 1 (a unit vector, not a cap);   */
/*        v = 0 -> no move; pos += brownian * displacement_rate                      */
/*   R42  Philox counter (id, step, 5): w0..w2 movement, w3 death;                    */
/*        (id, step, 6): w0 division; division axis as R13 (streams 3 + 4k)          */
/*   R43  growth as R28 (V += growth, d = 2 cbrt_det(V 0.75/pi)), division as R13      */
/*        (V/2 each, touching daughters, mother MOVED, daughter ADDED with age 0)     */
/*   R45  removal keeps the survivors' order; daughters follow the survivors in       */
/*        mother-id order with ids id_next + rank; ids are never reused               */
/* One pass in ascending id over agents carrying their post-mechanics state.         */
/* ------------------------------------------------------------------------------ */
typedef struct {
    double displacement_rate, growth, max_diameter, p_death, p_div;
    uint32_t min_age;
    uint64_t seed;
    uint32_t step;
} orc_onco_params;



/* Returns the new agent count (or -(required capacity) and leaves everything unchanged);
 * *id_next is advanced by the number of daughters. */
int64_t orc_onco_step(int64_t n, double *x, double *y, double *z, double *d, double *vol,
                      uint32_t *id, uint32_t *flags, uint32_t *age, int64_t capacity,
                      const orc_onco_params *p, int64_t *id_next)
{
    const double C = 0.75 / M_PI;
    /* ascending id order (ids are unique but not dense after removals) */
    orc_kv *kv = (orc_kv *)malloc(sizeof(orc_kv) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) { kv[i].key = (int64_t)id[i]; kv[i].idx = i; }
    qsort(kv, (size_t)n, sizeof(orc_kv), cmp_kv);
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) ord[i] = kv[i].idx;
    free(kv);
    uint8_t *dead = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    uint8_t *div = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    int64_t ndiv = 0, ndead = 0;
    /* first decide (draws only; nothing is modified before the capacity check) */
    for (int64_t k = 0; k < n; ++k) {
        int64_t i = ord[k];
        uint32_t w[4];
        philox_draw(p->seed, id[i], p->step, 5u, w);
        if (age[i] >= p->min_age && orc_u32(w[3]) < p->p_death) { dead[i] = 1; ++ndead; continue; }
        if (!(d[i] < p->max_diameter)) {
            uint32_t v[4];
            philox_draw(p->seed, id[i], p->step, 6u, v);
            if (orc_u32(v[0]) < p->p_div) { div[i] = 1; ++ndiv; }
        }
    }
    const int64_t nsurv = n - ndead, nnew = nsurv + ndiv;
    if (nnew > capacity || n > capacity) {
        free(ord); free(dead); free(div);
        return -(nnew > n ? nnew : n);
    }
    /* apply, in ascending id: Brownian move, age, growth or division */
    int64_t rank = 0;
    double *dx = (double *)malloc(sizeof(double) * (size_t)(ndiv > 0 ? ndiv : 1) * 3);
    double *dd = (double *)malloc(sizeof(double) * (size_t)(ndiv > 0 ? ndiv : 1) * 2);
    for (int64_t k = 0; k < n; ++k) {
        int64_t i = ord[k];
        if (dead[i]) continue;
        uint32_t w[4];
        philox_draw(p->seed, id[i], p->step, 5u, w);
        double vx = 2.0 * orc_u32(w[0]) - 1.0;
        double vy = 2.0 * orc_u32(w[1]) - 1.0;
        double vz = 2.0 * orc_u32(w[2]) - 1.0;
        double n2 = vx * vx + vy * vy + vz * vz;
        if (n2 > 0.0) {
            double nv = sqrt(n2);
            x[i] = x[i] + (vx / nv) * p->displacement_rate;
            y[i] = y[i] + (vy / nv) * p->displacement_rate;
            z[i] = z[i] + (vz / nv) * p->displacement_rate;
            if (p->displacement_rate != 0.0) flags[i] |= ORC_MOVED;
        }
        age[i] += 1u;
        if (d[i] < p->max_diameter) {
            double Vn = vol[i] + p->growth;
            double dn = 2.0 * orc_cbrt_det(Vn * C);
            if (dn > d[i]) flags[i] |= ORC_GREW;
            vol[i] = Vn;
            d[i] = dn;
        } else if (div[i]) {
            double Vh = vol[i] * 0.5;
            double r = orc_cbrt_det(Vh * C);
            double u[3];
            orc_division_axis(p->seed, id[i], p->step, u);
            double px = x[i], py = y[i], pz = z[i];
            x[i] = px - r * u[0];
            y[i] = py - r * u[1];
            z[i] = pz - r * u[2];
            dx[3 * rank + 0] = px + r * u[0];
            dx[3 * rank + 1] = py + r * u[1];
            dx[3 * rank + 2] = pz + r * u[2];
            dd[2 * rank + 0] = 2.0 * r;
            dd[2 * rank + 1] = Vh;
            vol[i] = Vh;
            d[i] = 2.0 * r;
            flags[i] |= ORC_MOVED;
            ++rank;
        }
    }
    /* removal: survivors keep their order */
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (dead[i]) continue;
        x[m] = x[i]; y[m] = y[i]; z[m] = z[i]; d[m] = d[i]; vol[m] = vol[i];
        id[m] = id[i]; flags[m] = flags[i]; age[m] = age[i];
        ++m;
    }
    /* daughters in mother-id order */
    for (int64_t r = 0; r < ndiv; ++r) {
        int64_t j = nsurv + r;
        x[j] = dx[3 * r + 0]; y[j] = dx[3 * r + 1]; z[j] = dx[3 * r + 2];
        d[j] = dd[2 * r + 0]; vol[j] = dd[2 * r + 1];
        id[j] = (uint32_t)(*id_next + r);
        flags[j] = ORC_ADDED;
        age[j] = 0u;
    }
    *id_next += ndiv;
    free(ord); free(dead); free(div); free(dx); free(dd);
    return nnew;
}

/* Initial ages for the oncology workload (reading R44): floor(u32(w0) * max_age) with
 * Philox (id, 0xFFFFFFFC, 2). */
void orc_init_ages(int64_t n, const uint32_t *id, uint64_t seed, uint32_t max_age, uint32_t *age)
{
    for (int64_t k = 0; k < n; ++k) {
        uint32_t w[4];
        philox_draw(seed, id[k], 0xFFFFFFFCu, 2u, w);
        age[k] = (uint32_t)floor(orc_u32(w[0]) * (double)max_age);
    }
}

/* ===================================================================== row f3
 * Delta-encoded + LZ4-compressed aura messages (sec. "Data Transfer Minimization",
 * P:6291-6356; evaluation P:6911-6937 with LZ4 [lz4]).  Readings R46-R51:
 *
 *   R46 the reference is a previous aura message held by sender and receiver, kept in
 *       ascending id order;
 *   R47 matching: slot r < nref carries the message agent whose id is
 *       ref.id[r], or a placeholder (presence bit 0); agents not in the reference
 *       follow at slots nref.. in message order;
 *   R48 "the difference" of a matched agent is the XOR of the IEEE bit patterns of
 *       x, y, z, d and of flags (lossless; id is implied by the slot); placeholders
 *       carry zeros; new agents carry their raw bits and their id;
 *   R49 payload layout: presence words, then the x, y, z, d columns over all
 *       nref + nnew slots each split into 8 byte planes, flags into 4 byte planes,
 *       then the ids of the new agents (little-endian);
 *   R50 LZ4 block format, payload cut into independent 1024-byte chunks; the match
 *       candidate of a position is the last earlier position with the same 11-bit
 *       hash of its next 4 bytes (h = (v * 2654435761) >> 21, every position enters
 *       the table); greedy parse, match >= 4 bytes, a match starts before n - 12 and
 *       ends by n - 5;
 *   R51 decoding restores the message in reference order (placeholders removed,
 *       P:6350-6352), then the new agents.
 * Stream: u32 magic 'BDA1', u32 chunk size, u64 nref, u64 nnew, u64 payload bytes,
 * u32 nchunks, u32 0, u32 compressed size per chunk, the chunks. */

#define ORC_LZ4_CHUNK 1024
#define ORC_LZ4_HBITS 11

static uint32_t rd32(const uint8_t *p)
{
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static int64_t lz4_put_len(uint8_t *dst, int64_t o, int64_t cap, int64_t L)
{
    while (L >= 255) {
        if (o >= cap) return -1;
        dst[o++] = 255;
        L -= 255;
    }
    if (o >= cap) return -1;
    dst[o++] = (uint8_t)L;
    return o;
}

/* One sequence: literals src[a, a+nlit), then (if mlen > 0) a match of mlen bytes at
 * distance off.  Returns the new output position or -1 (no room). */
static int64_t lz4_sequence(const uint8_t *src, int64_t a, int64_t nlit, int64_t off, int64_t mlen,
                            uint8_t *dst, int64_t o, int64_t cap)
{
    if (o >= cap) return -1;
    int64_t tok = o++;
    uint8_t t = (uint8_t)((nlit < 15 ? nlit : 15) << 4);
    if (nlit >= 15 && (o = lz4_put_len(dst, o, cap, nlit - 15)) < 0) return -1;
    if (o + nlit > cap) return -1;
    memcpy(dst + o, src + a, (size_t)nlit);
    o += nlit;
    if (mlen > 0) {
        if (o + 2 > cap) return -1;
        dst[o++] = (uint8_t)(off & 255);
        dst[o++] = (uint8_t)(off >> 8);
        int64_t m = mlen - 4;
        t |= (uint8_t)(m < 15 ? m : 15);
        if (m >= 15 && (o = lz4_put_len(dst, o, cap, m - 15)) < 0) return -1;
    }
    dst[tok] = t;
    return o;
}

/* R50: compress one block of n <= 65535 bytes.  Two passes, in this order:
 *   1. candidates: cand[p] = the last position q < p whose next 4 bytes hash to the
 *      same 11-bit bucket (every position of the block enters the table), or none;
 *   2. greedy parse from ip = 0: if ip < n - 12 and cand[ip] holds the same 4 bytes as
 *      ip, emit the literals since the last match and a match extended forward while
 *      the bytes agree and ip + len < n - 5, then continue after it; otherwise ip + 1.
 * Returns the compressed size or -1. */
int64_t orc_lz4_compress_block(const uint8_t *src, int64_t n, uint8_t *dst, int64_t cap)
{
    int32_t table[1 << ORC_LZ4_HBITS];
    for (int k = 0; k < (1 << ORC_LZ4_HBITS); ++k) table[k] = -1;
    int32_t *cand = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    for (int64_t p = 0; p < n; ++p) {
        cand[p] = -1;
        if (p + 4 > n) continue;
        uint32_t h = (uint32_t)(rd32(src + p) * 2654435761u) >> (32 - ORC_LZ4_HBITS);
        cand[p] = table[h];
        table[h] = (int32_t)p;
    }
    int64_t ip = 0, anchor = 0, o = 0;
    while (ip < n - 12) {
        int32_t ref = cand[ip];
        if (ref >= 0 && rd32(src + ref) == rd32(src + ip)) {
            int64_t len = 4;
            while (ip + len < n - 5 && src[ref + len] == src[ip + len]) ++len;
            o = lz4_sequence(src, anchor, ip - anchor, ip - ref, len, dst, o, cap);
            if (o < 0) { free(cand); return -1; }
            ip += len;
            anchor = ip;
        } else {
            ++ip;
        }
    }
    free(cand);
    o = lz4_sequence(src, anchor, n - anchor, 0, 0, dst, o, cap);
    return o;
}

/* LZ4 block decoder (format definition).  Returns the decoded size or -1 (malformed or
 * more than cap bytes). */
int64_t orc_lz4_decompress_block(const uint8_t *src, int64_t n, uint8_t *dst, int64_t cap)
{
    int64_t i = 0, o = 0;
    while (i < n) {
        uint8_t t = src[i++];
        int64_t nlit = t >> 4;
        if (nlit == 15) {
            uint8_t b;
            do {
                if (i >= n) return -1;
                b = src[i++];
                nlit += b;
            } while (b == 255);
        }
        if (i + nlit > n || o + nlit > cap) return -1;
        memcpy(dst + o, src + i, (size_t)nlit);
        i += nlit;
        o += nlit;
        if (i == n) break;  /* the last sequence has literals only */
        if (i + 2 > n) return -1;
        int64_t off = (int64_t)src[i] | ((int64_t)src[i + 1] << 8);
        i += 2;
        int64_t mlen = (t & 15) + 4;
        if ((t & 15) == 15) {
            uint8_t b;
            do {
                if (i >= n) return -1;
                b = src[i++];
                mlen += b;
            } while (b == 255);
        }
        if (off == 0 || off > o || o + mlen > cap) return -1;
        for (int64_t k = 0; k < mlen; ++k, ++o) dst[o] = dst[o - off]; /* may overlap */
    }
    return o;
}

static uint64_t bits64(double v)
{
    uint64_t b;
    memcpy(&b, &v, 8);
    return b;
}

static double from_bits64(uint64_t b)
{
    double v;
    memcpy(&v, &b, 8);
    return v;
}

static int64_t find_id(const uint32_t *ids, int64_t n, uint32_t id)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (ids[mid] < id) lo = mid + 1; else hi = mid;
    }
    return (lo < n && ids[lo] == id) ? lo : -1;
}

/* Payload size for nref reference slots and nnew new agents (R49). */
int64_t orc_aura_payload_size(int64_t nref, int64_t nnew)
{
    int64_t ns = nref + nnew;
    return 4 * ((nref + 31) / 32) + 4 * 8 * ns + 4 * ns + 4 * nnew;
}

/* R46-R49: the uncompressed payload of message (n agents) against the reference
 * (nref agents, ascending ids).  *nnew_out = agents not in the reference.  The payload
 * buffer must hold orc_aura_payload_size(nref, n) bytes.  Returns the payload size. */
int64_t orc_aura_payload(int64_t n, const double *x, const double *y, const double *z,
                         const double *d, const uint32_t *id, const uint32_t *flags,
                         int64_t nref, const double *rx, const double *ry, const double *rz,
                         const double *rd, const uint32_t *rid, const uint32_t *rflags,
                         uint8_t *out, int64_t *nnew_out)
{
    int64_t *slot_of = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t nnew = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t r = find_id(rid, nref, id[i]);
        slot_of[i] = r >= 0 ? r : nref + nnew++;
    }
    int64_t ns = nref + nnew, nw = (nref + 31) / 32;
    int64_t size = orc_aura_payload_size(nref, nnew);
    memset(out, 0, (size_t)size);
    uint8_t *pres = out;
    uint8_t *col = out + 4 * nw;             /* x, y, z, d: 8 planes of ns bytes each */
    uint8_t *fcol = col + 4 * 8 * ns;        /* flags: 4 planes */
    uint8_t *nid = fcol + 4 * ns;            /* ids of the new agents */
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = slot_of[i];
        const double mv[4] = {x[i], y[i], z[i], d[i]};
        uint64_t v[4];
        uint32_t f = flags[i];
        if (s < nref) {
            const double rv[4] = {rx[s], ry[s], rz[s], rd[s]};
            for (int c = 0; c < 4; ++c) v[c] = bits64(mv[c]) ^ bits64(rv[c]);
            f ^= rflags[s];
            pres[4 * (s / 32) + (s % 32) / 8] |= (uint8_t)(1u << (s % 8));
        } else {
            for (int c = 0; c < 4; ++c) v[c] = bits64(mv[c]);
            int64_t j = s - nref;
            for (int b = 0; b < 4; ++b) nid[4 * j + b] = (uint8_t)(id[i] >> (8 * b));
        }
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 8; ++b) col[(int64_t)(8 * c + b) * ns + s] = (uint8_t)(v[c] >> (8 * b));
        for (int b = 0; b < 4; ++b) fcol[(int64_t)b * ns + s] = (uint8_t)(f >> (8 * b));
    }
    free(slot_of);
    *nnew_out = nnew;
    return size;
}

/* R51: the message back from a payload and the reference; returns its size n
 * (reference-order survivors, then the new agents). */
int64_t orc_aura_unpayload(const uint8_t *in, int64_t nref, int64_t nnew, const double *rx,
                           const double *ry, const double *rz, const double *rd,
                           const uint32_t *rid, const uint32_t *rflags, double *x, double *y,
                           double *z, double *d, uint32_t *id, uint32_t *flags)
{
    int64_t ns = nref + nnew, nw = (nref + 31) / 32;
    const uint8_t *pres = in, *col = in + 4 * nw, *fcol = col + 4 * 8 * ns, *nid = fcol + 4 * ns;
    int64_t m = 0;
    for (int64_t s = 0; s < ns; ++s) {
        int present = s >= nref || ((pres[4 * (s / 32) + (s % 32) / 8] >> (s % 8)) & 1);
        if (!present) continue;
        uint64_t v[4] = {0, 0, 0, 0};
        uint32_t f = 0;
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 8; ++b) v[c] |= (uint64_t)col[(int64_t)(8 * c + b) * ns + s] << (8 * b);
        for (int b = 0; b < 4; ++b) f |= (uint32_t)fcol[(int64_t)b * ns + s] << (8 * b);
        if (s < nref) {
            const double rv[4] = {rx[s], ry[s], rz[s], rd[s]};
            for (int c = 0; c < 4; ++c) v[c] ^= bits64(rv[c]);
            f ^= rflags[s];
            id[m] = rid[s];
        } else {
            int64_t j = s - nref;
            id[m] = (uint32_t)nid[4 * j] | ((uint32_t)nid[4 * j + 1] << 8) |
                    ((uint32_t)nid[4 * j + 2] << 16) | ((uint32_t)nid[4 * j + 3] << 24);
        }
        x[m] = from_bits64(v[0]);
        y[m] = from_bits64(v[1]);
        z[m] = from_bits64(v[2]);
        d[m] = from_bits64(v[3]);
        flags[m] = f;
        ++m;
    }
    return m;
}

/* R50: the stream of a payload (header, sizes, LZ4 chunks).  Returns its size or -1. */
int64_t orc_aura_compress(const uint8_t *payload, int64_t size, int64_t nref, int64_t nnew,
                          uint8_t *out, int64_t cap)
{
    int64_t nch = (size + ORC_LZ4_CHUNK - 1) / ORC_LZ4_CHUNK;
    int64_t hdr = 40 + 4 * nch;
    if (cap < hdr) return -1;
    uint32_t h32[2] = {0x31414442u, ORC_LZ4_CHUNK};
    uint64_t h64[3] = {(uint64_t)nref, (uint64_t)nnew, (uint64_t)size};
    uint32_t t32[2] = {(uint32_t)nch, 0u};
    memcpy(out, h32, 8);
    memcpy(out + 8, h64, 24);
    memcpy(out + 32, t32, 8);
    int64_t o = hdr;
    for (int64_t c = 0; c < nch; ++c) {
        int64_t a = c * ORC_LZ4_CHUNK, len = size - a < ORC_LZ4_CHUNK ? size - a : ORC_LZ4_CHUNK;
        int64_t k = orc_lz4_compress_block(payload + a, len, out + o, cap - o);
        if (k < 0) return -1;
        uint32_t k32 = (uint32_t)k;
        memcpy(out + 40 + 4 * c, &k32, 4);
        o += k;
    }
    return o;
}

/* Inverse of orc_aura_compress: writes the payload, returns its size (or -1) and the
 * header's nref / nnew. */
int64_t orc_aura_decompress(const uint8_t *in, int64_t n, uint8_t *payload, int64_t cap,
                            int64_t *nref, int64_t *nnew)
{
    if (n < 40) return -1;
    uint32_t h32[2], t32[2];
    uint64_t h64[3];
    memcpy(h32, in, 8);
    memcpy(h64, in + 8, 24);
    memcpy(t32, in + 32, 8);
    if (h32[0] != 0x31414442u || h32[1] != ORC_LZ4_CHUNK) return -1;
    int64_t size = (int64_t)h64[2], nch = t32[0];
    if (size > cap || nch != (size + ORC_LZ4_CHUNK - 1) / ORC_LZ4_CHUNK || n < 40 + 4 * nch) return -1;
    int64_t o = 40 + 4 * nch;
    for (int64_t c = 0; c < nch; ++c) {
        uint32_t k;
        memcpy(&k, in + 40 + 4 * c, 4);
        int64_t a = c * ORC_LZ4_CHUNK, len = size - a < ORC_LZ4_CHUNK ? size - a : ORC_LZ4_CHUNK;
        if (o + k > n) return -1;
        if (orc_lz4_decompress_block(in + o, k, payload + a, len) != len) return -1;
        o += k;
    }
    *nref = (int64_t)h64[0];
    *nnew = (int64_t)h64[1];
    return size;
}
