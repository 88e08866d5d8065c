/*
 * bdm.h -- C ABI of the B200-native BioDynaMo/TeraAgent mechanics hot path
 * (arXiv 2503.10796).  Implemented by paper_2503_10796_b200/libbdm.so (sm_100a).
 *
 * Citations "P:a-b" are lines of PAPER.md (the thesis' LaTeX source); the section,
 * equation or algorithm label is given alongside.  "Rn" refers to the numbered
 * readings in DESIGN.md section 3 (where the paper is silent or ambiguous).
 *
 * Conventions for every entry point
 *   - All agent-array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     unless the entry point's name ends in _host.  Arrays are structure-of-arrays,
 *     indexed [0, n), 8-byte aligned; they are owned by the caller.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *     Every call only enqueues work on `stream` unless documented as synchronizing.
 *   - The library owns its workspace (allocated in bdm_create / grown on demand in
 *     bdm_grid_build and bdm_reserve); nothing is allocated inside bdm_mech_step.
 *   - Every call returns a bdm_status; no C++ exception crosses the ABI.
 *     bdm_last_error() returns a thread-local message for the last failure.
 *   - Device-side conditions (grid-slot capacity exceeded, non-finite positions)
 *     are latched in device memory; the kernels of the affected step become no-ops
 *     (the caller's arrays are left exactly as they were) and bdm_sync() reports
 *     the condition.  The caller may then bdm_reserve() and re-issue the step.
 *   - n == 0 is valid and every compute call is a no-op for it.
 */
#ifndef BDM_H
#define BDM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BDM_OK = 0,
    BDM_EINVAL = -1,      /* bad argument (null pointer, n > capacity, radius < 0, ...) */
    BDM_ECAPACITY = -2,   /* a library or caller capacity is too small; see bdm_last_error */
    BDM_ECUDA = -3,       /* CUDA runtime error (possibly from an earlier async launch) */
    BDM_ENCCL = -4,       /* NCCL missing or a collective failed (bdm_last_error)     */
    BDM_ENOTFINITE = -5,  /* a position was NaN/Inf */
    BDM_ENOTIMPL = -6     /* feature not implemented in this build */
} bdm_status;

/* Agent flag bits (R8, R31; static-agent conditions of P:4941-4946).  Set by a
 * step, read by the next step. */
#define BDM_FLAG_MOVED 0x1u   /* displacement != 0 in the last step (condition i)    */
#define BDM_FLAG_GREW 0x2u    /* diameter increased in the last step (condition ii)  */
#define BDM_FLAG_ADDED 0x4u   /* created in the last step (condition iii); initial
                                 agents carry it so nobody is static at step 0     */
#define BDM_FLAG_STATIC 0x8u  /* the force was skipped in the last step             */
#define BDM_FLAG_NNZ_SHIFT 4  /* bits 4-5: #non-zero neighbour forces, saturating at
                                 2 (condition iv)                                   */

/* Structure-of-arrays agent storage (D01/D02 of SURVEY).  Caller-owned
 * device memory, `capacity` elements each.  A mechanics step reorders all arrays
 * (agents travel with their id), see bdm_mech_step. */
typedef struct {
    int64_t n;            /* live agents                                           */
    int64_t capacity;     /* allocated elements of every array                     */
    double *x, *y, *z;    /* centre of mass [um or m]                              */
    double *diameter;     /* sphere diameter d = 2r                                 */
    double *volume;       /* nullable (growth/division only)                       */
    uint32_t *id;         /* immutable global agent id (A50)                       */
    uint32_t *flags;      /* BDM_FLAG_* bits                                       */
    uint8_t *state;       /* nullable (SIR only): 0 S, 1 I, 2 R                    */
} bdm_agents;

/* Parameters of one mechanics step. */
typedef struct {
    double k, gamma;           /* Eq. 4.1 coefficients, 2 and 1 in the paper */
    double dt;                 /* displacement = dt * sum of forces (R6)                    */
    double max_displacement;   /* cap on |displacement| per step (R6)                       */
    double force_threshold;    /* move only if |F| > threshold (R7)            */
    double radius;             /* interaction radius; <= 0: largest diameter  */
    int32_t detect_static;     /* 1: skip the force of static agents (sec:static-agents)    */
    int32_t boundary;          /* 0 open (P:2671 (i)), 1 closed = clamp to [lo, hi],       */
                               /* 2 toroidal = the periodic cube [0, hi[0])^3 (R52)         */
    double lo[3], hi[3];       /* closed-boundary box; toroidal: lo = 0, hi = (side,side,side) */
    uint64_t seed;             /* Philox key for steps that draw random numbers            */
    uint32_t step;             /* iteration number (Philox counter word)                    */
    uint32_t collect_stats;    /* 1: count candidates/neighbours/contacts (costs atomics)  */
} bdm_params;

/* Per-step work counters (sums over the agents of the step). */
typedef struct {
    int64_t cand;      /* candidates examined in the 27 boxes (force loop only)     */
    int64_t nbr;       /* of which within the interaction radius (D <= R^2)         */
    int64_t cont;      /* of which in contact (overlap delta > 0)                   */
    int64_t n_static;  /* agents whose force was skipped                           */
    int64_t n_moved;   /* agents with a non-zero displacement                      */
    int64_t launches;  /* kernels launched by this context since bdm_create (cumulative,
                          host-side count; independent of collect_stats)            */
} bdm_stats;

/* Geometry of the last grid build (a1 of SURVEY section 8(a)). */
typedef struct {
    double R, L;             /* interaction radius and box edge L = R(1+2^-20) (R5)  */
    double origin[3];        /* per-axis minimum of the positions (R12)              */
    double upper[3];         /* per-axis maximum                                     */
    int64_t dims[3];         /* boxes per axis                                        */
    int64_t nslots;          /* blocked-Morton key slots = ceil(dims/4)^3 * 64 (R32)   */
    int64_t slot_capacity;   /* allocated slots                                       */
} bdm_grid_info;

/* Diffusion grid (reading R34): nx*ny*nz points of a substance,
 * fp64, point (i,j,k) stored at index i + nx*(j + ny*k) (x fastest), the centre of the
 * cell [lo + i*dx, lo + (i+1)*dx) x [..dy..) x [..dz..).  Values outside the grid are 0
 * ("substances diffuse out of the simulation space"). */
typedef struct {
    int64_t nx, ny, nz;      /* points per axis (nx*ny < 2^31, nz < 2^31)             */
    double lo[3];            /* lower corner of cell (0,0,0)                          */
    double dx, dy, dz;       /* cell edge per axis (> 0)                              */
} bdm_grid3;

typedef struct bdm_ctx *bdm_handle;

/* Create a library context on CUDA device `device` with workspace for up to
 * `max_agents` agents (grown automatically by bdm_grid_build if exceeded).
 * Synchronizing.  Errors: BDM_EINVAL (max_agents < 0, bad device), BDM_ECUDA. */
bdm_status bdm_create(bdm_handle *out, int device, int64_t max_agents);

/* Caller-supplied device allocator (the caller, e.g. torch's caching
 * allocator, owns the device memory pool; the paper's engine likewise takes its agent
 * memory from one pool allocator).  `alloc` returns a device pointer to at
 * least `bytes` bytes aligned to 256 B, usable on `stream` (NULL: any stream, the
 * device is idle), or NULL on failure; `release` takes a pointer `alloc` returned.
 * `user` is passed through unchanged. */
typedef void *(*bdm_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*bdm_free_fn)(void *ptr, void *stream, void *user);

/* bdm_create with the workspace sized for `max_agents` local agents plus `max_ghosts`
 * aura agents (bdm_grid_build sorts locals and ghosts together, section 8(e)) and,
 * when `alloc`/`release` are both non-NULL, every per-agent, grid (box starts, scan
 * sums) and slab-exchange buffer taken from and returned to them: at creation, at
 * capacity growth and in bdm_destroy, never inside a step of steady size.  The few
 * context scalars (< 1 KB), the dense kernel's scratch and the first-use workspaces of
 * the SIR, oncology and aura-codec rows use cudaMalloc.  The callbacks must stay valid
 * until bdm_destroy returns and are called from the thread that calls the library.
 * Synchronizing.  Errors: BDM_EINVAL (negative sizes, bad device, only one of the two
 * callbacks given), BDM_ECAPACITY (`alloc` returned NULL), BDM_ECUDA. */
bdm_status bdm_create_ex(bdm_handle *out, int device, int64_t max_agents, int64_t max_ghosts,
                         bdm_alloc_fn alloc, bdm_free_fn release, void *user);

/* Free the context and its workspace.  Synchronizing.  NULL is a no-op. */
bdm_status bdm_destroy(bdm_handle h);

/* Thread-local description of the last error ("" if none). */
const char *bdm_last_error(void);

/* Library version string ("bdm <semver> sm_100a"). */
const char *bdm_version(void);

/* Uniform-in-cube population (ModelInitializer) with the per-agent
 * counter-based PRNG the paper proposes: for agent id = id0 + k,
 * Philox4x32-10 with key = seed and counter (id_lo, id_hi, w, 2) gives
 * x, y from w = 0xFFFFFFFF, z from w = 0xFFFFFFFE, and, if d_random, the diameter
 * d = d_lo + d_width * u53 from w = 0xFFFFFFFD (R22, R23, R29); else d = d_lo.
 * Writes agents [0, n) of `a` (a->n is set to n) with flags = BDM_FLAG_ADDED.
 * Errors: BDM_EINVAL if n > a->capacity or a required pointer is NULL. */
bdm_status bdm_init_spheres(bdm_handle h, bdm_agents *a, int64_t id0, int64_t n,
                            uint64_t seed, double side, double d_lo, double d_width,
                            int32_t d_random, void *stream);

/* Grid build ("Environment Search" P:2584-2598, sec:grid
 * P:4487-4530, agent sorting sec:load-balancing P:4720-4838):
 *   a1  R = radius > 0 ? radius : max_i d_i; L = R(1+2^-20); origin = per-axis min;
 *       dims = floor((max - origin)/L) + 1                               (R5, R12)
 *   a2  box b = floor((x - origin)/L); blocked-Morton key (4^3 tiles, row-major
 *       tiles, 3-D Morton inside, x in the lowest bit)                   (R32)
 *   a3  box start/length by an exclusive scan of per-slot counts (replaces the
 *       paper's timestamped array linked list)
 *   a4  counting sort by key, ascending id inside a box, gather of the SoA into
 *       the library's sorted workspace.
 * `ghosts` (nullable) are read-only agents owned by a neighbouring rank (aura,
 * P:6083-6106): they enter the grid (and the canonical order) but are never
 * updated; the following bdm_mech_step writes only the local agents.
 * With a frame set by bdm_set_frame, the origin and R come from the frame (the
 * global grid of a multi-GPU run) and only the lattice extent is local.
 * The first call for a given context synchronizes once to size the slot array;
 * later calls are asynchronous.  Errors: BDM_EINVAL, BDM_ECUDA. */
bdm_status bdm_grid_build(bdm_handle h, const bdm_agents *a, const bdm_agents *ghosts,
                          double radius, void *stream);

/* Mechanics step over the grid of the preceding bdm_grid_build on the same agents
 * (rows a5-a9: MechanicalForcesOp + BoundSpaceOp; Eq. 4.1/4.2
 * P:2720-2741; static-agent skip sec:static-agents P:4920-4965).  Copy (Jacobi)
 * semantics (R11).  For every agent i, in the canonical order of R9
 * (27 boxes in (dz,dy,dx) lexicographic order, ascending id inside a box):
 *   D = fma(dz,dz, fma(dy,dy, dx*dx)), (dx,dy,dz) = x_i - x_j; neighbour iff D <= R^2
 *   dist = sqrt(D); delta = (r_i + r_j) - dist; if delta > 0 and dist > 0:
 *     rbar = r_i r_j/(r_i + r_j); F_N = k delta - gamma sqrt(rbar delta);
 *     F_i = fma(F_N/dist, x_i - x_j, F_i) per component
 *   displacement = dt F_i if |F_i|^2 > threshold^2 else 0, capped at
 *   max_displacement; x_i += displacement; boundary (open: no-op; closed: clamp;
 *   toroidal: x = fmod(x, side), + side if negative -- Alg. 9's wrap, R20).
 * Toroidal (boundary 2, P:2671 (iii), reading R52): the grid is the periodic lattice of
 * [0, side)^3, D = floor(side / R) >= 3 boxes of edge side / D per axis; the 27 boxes
 * wrap modulo D (same canonical order) and (dx,dy,dz) is the minimum image (+-side
 * beyond side/2).  Only bdm_step builds that grid (the reference formulation runs).
 * Static agents (R8) skip the force: displacement 0, nnz carried.
 * On return (stream order) the caller's arrays x,y,z,diameter,id,flags hold the
 * new state in the grid's sorted order (key, then id): a permutation of the input
 * (or, on builds that option "sort_every" leaves in place, in the input order).
 * Errors: BDM_EINVAL (no matching grid build, bad params, a toroidal step without its
 * grid; deferred: side < 3 R), BDM_ECUDA. */
bdm_status bdm_mech_step(bdm_handle h, bdm_agents *a, const bdm_params *p, void *stream);

/* Convenience: bdm_grid_build(a, NULL, p->radius) then bdm_mech_step(a, p); with
 * boundary 2 the build is on the torus (lo must be 0 and hi a cube, else BDM_EINVAL). */
bdm_status bdm_step(bdm_handle h, bdm_agents *a, const bdm_params *p, void *stream);

/* End-to-end step on HOST arrays (the e2e entry point): copies the n agents of
 * `host_in` to the device arrays `dev` (host->device), runs bdm_step, copies the
 * new state back into `host_out` (device->host) and synchronizes `stream`.
 * host_in may equal host_out.  In place (the same diameter and id arrays) on a step
 * that keeps the input order (option "sort_every"), only x, y, z and flags are copied
 * back: a mechanics step does not change d or id.  Host arrays should be pinned for
 * full bandwidth.
 * Errors: as bdm_step, plus deferred device conditions (as bdm_sync). */
bdm_status bdm_step_host(bdm_handle h, const bdm_agents *host_in, bdm_agents *host_out,
                         bdm_agents *dev, const bdm_params *p, void *stream);

/* K end-to-end steps on the HOST state `host` (in place): every step copies the n
 * agents host -> device (x, y, z, diameter, id, flags into `dev`), runs bdm_step and
 * copies the new state device -> host (x, y, z, flags; diameter and id too unless the
 * step kept the input order, option "sort_every").  Pipelined: the arrays are split
 * into `chunks` (1..64) index ranges, and chunk c of step k+1 is uploaded as soon as
 * chunk c of step k has come down, so downloads and uploads overlap on PCIe (two copy
 * streams next to `stream`).  Host arrays must be pinned for the overlap.  Returns
 * after the last download (synchronizes).  Errors: as bdm_step_host. */
bdm_status bdm_run_host(bdm_handle h, bdm_agents *host, bdm_agents *dev, const bdm_params *p,
                        int32_t steps, int32_t chunks, void *stream);

/* Growth and division with add-compaction (Alg. 4 control flow
 * "grow while below the maximum size, else divide", with division
 * probability 1; Cell::Divide; parallel addition).  Reads
 * the start-of-step volume (R15) of every agent i in [0, n):
 *   V < v_max:  V += growth; d = 2 cbrt_det(V * 0.75/pi) (R28); GREW if d increased
 *   else:       V/2 for mother and daughter, r' = cbrt_det(V/2 * 0.75/pi), axis u from
 *               Philox(seed, id, p->step, stream 3 + 4k) by rejection (R13); mother
 *               at x - r'u (MOVED), daughter at x + r'u (ADDED) with id n + rank and
 *               stored at index n + rank, rank = position among the dividers in id
 *               order.  Requires volume != NULL and ids exactly 0..n-1.
 * Usually called right after bdm_mech_step (positions are post-mechanics).  Writes
 * the new count to *n_out_host (pinned host memory, asynchronously; valid after the
 * stream synchronizes); a->n is NOT updated.  If n + #dividers > capacity nothing is
 * modified, *n_out_host = -(required capacity) and bdm_sync reports BDM_ECAPACITY.
 * An id >= n (ids not dense) is detected on the device: nothing is modified,
 * *n_out_host = n and bdm_sync reports BDM_EINVAL.
 * Errors: BDM_EINVAL (no volume array, growth < 0, v_max <= 0). */
bdm_status bdm_grow_divide(bdm_handle h, bdm_agents *a, const bdm_params *p, double growth,
                           double v_max, int64_t *n_out_host, void *stream);

/* SIR epidemiology step (Algorithms 7-9) on point
 * agents (x, y, z, state; id nullable = index) in the periodic cube [0, side)^3, in
 * place.  For every agent, from the start-of-step snapshot (R16-R22):
 *   w = Philox(seed, (id, p->step, 0)); if S and u32(w3) < p_inf and an agent that was
 *   infected at the start of the step lies within `radius` (minimum image): I;
 *   if I and u32(Philox(seed, (id, p->step, 1)).w0) < p_rec: R;
 *   v = 2 u32(w0..w2) - 1, v /= |v| if |v| > 1; x = wrap(x + v) with Alg. 9's
 *   el = fmod(el, side); if el < 0: el = side + el.
 * No fused multiply-add.  Needs 3 <= side/radius < 8193 (boxes per axis; the
 * infected-index hash keys hold the box index in 40 bits), else BDM_EINVAL.  If
 * counts_host (pinned, 4 int64)
 * is non-NULL it receives S, I, R after the step and the number of new infections
 * (asynchronously).  The infected index holds up to max(65536, n/16) agents (option
 * "sir_index_capacity"); beyond that the step is a no-op and bdm_sync reports
 * BDM_ECAPACITY.  Errors: BDM_EINVAL. */
bdm_status bdm_sir_step(bdm_handle h, bdm_agents *a, const bdm_params *p, double side,
                        double radius, double p_inf, double p_rec, int64_t *counts_host,
                        void *stream);

/* ---- extracellular diffusion, secretion, chemotaxis -------- */

/* Eq. 4.3 (eq:centraldiff): one explicit step from the device grid u_in to
 * u_out (layout bdm_grid3; distinct buffers, the caller alternates them over steps).
 * Per point, in this order and without fused multiply-add (R35):
 *   v = u*(1 - mu*dt)
 *   v = v + cx*((u[i+1] - 2u) + u[i-1]),  cx = (nu*dt)/(dx*dx); then the y and z terms,
 * with 0 for neighbours outside the grid (R34).  The explicit scheme is stable for
 * 2(cx + cy + cz) <= 1 - mu*dt; the call does not check it.  Asynchronous on stream.
 * Errors: BDM_EINVAL (NULL pointers, u_in == u_out, non-positive spacing). */
bdm_status bdm_diffuse(bdm_handle h, const double *u_in, double *u_out, const bdm_grid3 *g,
                       double nu, double mu, double dt, void *stream);

/* Alg. secretion_module: every agent i < a->n with type[i] == type_sel adds
 * q to the grid point of the cell containing (x, y, z)_i; cells are floor((p - lo)/d),
 * clamped to the grid (R36).  type is a device u8 array of a->n entries.  The result is
 * independent of the order of the additions because every addend is the same q.
 * Errors: BDM_EINVAL. */
bdm_status bdm_secrete(bdm_handle h, const bdm_agents *a, const uint8_t *type, int32_t type_sel,
                       double q, double *u, const bdm_grid3 *g, void *stream);

/* Alg. chemotaxis_module: every agent with type[i] == type_sel moves, in
 * place, by weight * GetNormalizedGradient: the central difference at its cell,
 * g_a = (u[+1] - u[-1]) / (2 d_a) with 0 outside the grid (R37), divided by
 * sqrt((gx*gx + gy*gy) + gz*gz) (no move for a zero gradient); p_a = p_a + weight*g_a
 * (R38).  Only x, y, z are read and written.  Errors: BDM_EINVAL. */
bdm_status bdm_chemotaxis(bdm_handle h, bdm_agents *a, const uint8_t *type, int32_t type_sel,
                          double weight, const double *u, const bdm_grid3 *g, void *stream);

/* ---- oncology behaviour with agent removal ------------------ */

/* Alg. 4 (algo:tumor_growth_module); values of Table 4.2 per
 * step of 1 h: displacement_rate 0.005 um, growth 42 um^3, p_div 0.0215, p_death 0.033,
 * min_age 87.  max_diameter is not given by the paper (reading R43: 14 um). */
typedef struct {
    double displacement_rate;  /* Brownian step length per step                       */
    double growth;             /* volume added per step while d < max_diameter        */
    double max_diameter;       /* growth below it, else division with p_div            */
    double p_death;            /* per step, for agents with age >= min_age             */
    double p_div;              /* per step, for agents with d >= max_diameter          */
    uint32_t min_age;          /* steps                                                */
    uint64_t seed;
    uint32_t step;
} bdm_onco_params;

/* One oncology behaviour pass with removal over agents carrying their post-mechanics
 * state (call after bdm_step; reading R40).  For every agent, in any memory order, with
 * Philox(seed, (id, step, 5)) = w and (id, step, 6) = v (R42):
 *   b = 2 u32(w0..w2) - 1, x += (b / |b|) * displacement_rate (R41; b = 0: no move);
 *   if age >= min_age and u32(w3) < p_death: removed;
 *   else age += 1 and, if d < max_diameter, V += growth, d = 2 cbrt_det(V 0.75/pi) (R28),
 *   else if u32(v0) < p_div: Cell::Divide as bdm_grow_divide (R13).
 * Removal keeps the survivors' relative order; daughters follow them in mother-id order
 * with ids id_next + rank (R45); ids are never reused.  Requires x, y, z, diameter,
 * volume, id (all < id_next, unique) and flags.  age is a device u32 property table
 * indexed by id (age_cap entries; the mechanics step reorders the SoA, ids travel with
 * it): read and incremented for every survivor, 0 for a daughter.  out_host (pinned, 2
 * int64) receives the new n and the new id_next, asynchronously; a->n is NOT updated.
 * If the new population exceeds a->capacity or the new id_next exceeds age_cap nothing
 * is modified, out_host[0] = -(required capacity) and bdm_sync reports BDM_ECAPACITY.
 * Errors: BDM_EINVAL. */
bdm_status bdm_onco_step(bdm_handle h, bdm_agents *a, uint32_t *age, int64_t age_cap,
                         const bdm_onco_params *p, int64_t id_next, int64_t *out_host,
                         void *stream);

/* ---- multi-GPU x-slabs (TeraAgent partitioning P:6058-6081,
 * aura update P:6083-6106, agent migration P:6116-6126).
 *
 * Rank r of N owns the static x-slab [slab_lo, slab_hi) (rank 0 unbounded below,
 * rank N-1 above: every agent has exactly one owner, R24).  One bdm_aura_exchange per
 * step, before bdm_grid_build(local, ghosts), does on `stream`, with ONE host
 * synchronization (for the received counts):
 *   - the global grid frame: element-wise MIN all-reduce of (min x, min y, min z,
 *     -max d) of the local agents; the following grid builds use it (R12), so every
 *     rank's box lattice and canonical order are those of the undivided run;
 *   - migration: agents with x < slab_lo go to rank r-1, x >= slab_hi to rank r+1
 *     and leave `local` (removal by refilling their slots from the end, Fig. 5.1);
 *   - aura: staying agents with x < slab_lo + R' go to rank r-1 and x >= slab_hi - R'
 *     to rank r+1, R' = R (1 + 2^-20) (R24), R = `radius` of bdm_dist_init or, if
 *     that is <= 0, the global largest diameter -- computed on the device;
 *   - local <- kept agents + arrivals; ghosts <- the neighbours' aura + this rank's own
 *     leavers (they belong to the neighbour now and lie at the shared border).
 * local->n and ghosts->n are updated.  The agent order in `local` changes (no result
 * depends on it, R32).  Buffers for sending and receiving are the library's
 * (persistent, grown geometrically; nothing is allocated in a step of steady size).
 * Precondition: agents move less than (slab width - R') per step.
 * Errors: BDM_EINVAL (arguments, no bdm_dist_init), BDM_ENCCL (NCCL missing or a
 * collective failed), BDM_ECUDA, BDM_ECAPACITY (local or ghosts too small for the
 * arrivals: the received agents are kept by the library, local->n = the kept
 * count; bdm_aura_pending gives the sizes needed, then grow the arrays (keeping
 * their contents) and call bdm_aura_finish). */
#define BDM_PACK_MIGRATE 1  /* x < lo -> left, x >= hi -> right; leavers removed        */
#define BDM_PACK_AURA 2     /* x < lo + margin -> left, x >= hi - margin -> right; copy */

/* A new NCCL unique id (128 bytes) for bdm_dist_init; rank 0 makes it, the caller
 * broadcasts it (e.g. torch.distributed).  The library links no NCCL: it resolves the
 * nine entry points it uses from the process's libnccl.so.2 (torch's, if loaded), or
 * from the library named by the environment variable BDM_NCCL_LIB when that is set
 * (another NCCL build; the tests' stand-in).  Errors: BDM_ENCCL (no such library). */
bdm_status bdm_nccl_unique_id(uint8_t id[128]);

/* Join the N-rank x-slab group (NCCL communicator from the 128-byte unique id; N = 1
 * needs no NCCL).  radius > 0 fixes R for the aura margin, else R = max diameter.
 * Collective over the N ranks (blocks until all joined).  One rank per GPU. */
bdm_status bdm_dist_init(bdm_handle h, const uint8_t nccl_unique_id[128], int32_t rank,
                         int32_t nranks, double slab_lo, double slab_hi, double radius);

/* One step's frame + migration + aura exchange (see above). */
bdm_status bdm_aura_exchange(bdm_handle h, bdm_agents *local, bdm_agents *ghosts, void *stream);

/* Virtual slabs (tests on one GPU): N contexts of one process on one device form a
 * group; bdm_aura_exchange_virtual does the exchange for all of them at once (device
 * copies instead of NCCL), with the same semantics and one synchronization.
 * slab_lo/slab_hi: N bounds each (outer bounds ignored, unbounded). */
bdm_status bdm_dist_init_virtual(bdm_handle *hs, int32_t nranks, const double *slab_lo,
                                 const double *slab_hi, double radius);
bdm_status bdm_aura_exchange_virtual(bdm_handle *hs, int32_t nranks, bdm_agents *locals,
                                     bdm_agents *ghosts, void *stream);

/* After BDM_ECAPACITY from an exchange: need[0] = local capacity needed, need[1] =
 * ghost capacity needed (0, 0 when nothing is pending). */
bdm_status bdm_aura_pending(bdm_handle h, int64_t need[2]);
/* Completes a pending exchange into the (grown) arrays; local->n must be the kept
 * count the exchange left. */
bdm_status bdm_aura_finish(bdm_handle h, bdm_agents *local, bdm_agents *ghosts, void *stream);

/* The device halves used by the Python reference protocol (slabs.py, CPU tests):
 * the local frame, packing and appending. */
#define BDM_PACK_MIGRATE 1  /* x < lo -> left, x >= hi -> right; leavers removed        */
#define BDM_PACK_AURA 2     /* x < lo + margin -> left, x >= hi - margin -> right; copy */

/* Local frame of `a`: frame_dev[0..2] = exact per-axis minimum of x, y, z and
 * frame_dev[3] = -(largest diameter) (device memory, 4 doubles).  An element-wise
 * MIN all-reduce of the ranks' frames gives the global frame (R12: origin = minimum
 * corner, R = largest diameter).  n == 0 gives (+inf, +inf, +inf, +inf). */
bdm_status bdm_local_frame(bdm_handle h, const bdm_agents *a, double *frame_dev, void *stream);

/* Use the global frame at frame_dev (device, 4 doubles as above; must stay valid) for
 * subsequent grid builds, or NULL to return to the local frame (single GPU). */
bdm_status bdm_set_frame(bdm_handle h, const double *frame_dev);

/* Pack agents of `a` for the slab [lo, hi) into the caller's send buffers
 * to_left / to_right (device SoA; x, y, z, diameter, id, flags, volume if both have
 * it), in no particular order (no result depends on the order of agents, R32).
 * BDM_PACK_MIGRATE: x < lo -> left, x >= hi -> right, and the
 * leavers are removed from `a`: the remaining agents above the new count move into the
 * leavers' slots (the paper's parallel removal; the order of the agents in
 * `a` changes, which no result depends on).  BDM_PACK_AURA:
 * x < lo + margin -> left, x >= hi - margin -> right (copies; `a` unchanged).
 * counts_host (pinned, 3 int64, asynchronous) receives #left, #right, #remaining;
 * to_left->n, to_right->n and a->n are NOT updated.  If a send buffer is too small
 * nothing is modified, the counts are negated and bdm_sync reports BDM_ECAPACITY. */
bdm_status bdm_pack_slab(bdm_handle h, bdm_agents *a, double lo, double hi, double margin,
                         int32_t what, bdm_agents *to_left, bdm_agents *to_right,
                         int64_t *counts_host, void *stream);

/* Append src[0, src->n) at dst[dst->n, ...) (device to device) and add src->n to
 * dst->n.  Errors: BDM_ECAPACITY if dst->n + src->n > dst->capacity. */
bdm_status bdm_append(bdm_handle h, bdm_agents *dst, const bdm_agents *src, void *stream);

/* Synchronize `stream` and report latched device conditions: BDM_ECAPACITY (grid
 * slots exceeded; bdm_get_grid_info gives the needed nslots), BDM_ENOTFINITE, or a
 * CUDA error.  Clears the latched condition. */
bdm_status bdm_sync(bdm_handle h, void *stream);

/* Ensure at least `nslots` grid slots and `max_agents` agents of workspace.
 * Synchronizing. */
bdm_status bdm_reserve(bdm_handle h, int64_t max_agents, int64_t nslots);

/* Work counters of the last step issued with collect_stats = 1.  Synchronizes. */
bdm_status bdm_get_stats(bdm_handle h, bdm_stats *out);

/* Geometry of the last grid build.  Synchronizes. */
bdm_status bdm_get_grid_info(bdm_handle h, bdm_grid_info *out);

/* Test hook: all ordered neighbour pairs (id_i << 32 | id_j), j != i, D_ij <= R^2
 * (R = radius > 0 ? radius : max diameter), enumerated through the grid (builds
 * one, which replaces the grid of any previous bdm_grid_build).  Writes at most
 * `cap` pairs (unordered) to the device array `pairs` and the total count to
 * *count_host.  Synchronizing.  Returns BDM_ECAPACITY if count > cap. */
bdm_status bdm_neighbor_pairs(bdm_handle h, const bdm_agents *a, double radius,
                              uint64_t *pairs, int64_t cap, int64_t *count_host,
                              void *stream);

/* Tuning/diagnostic options (host-side, take effect at the next launch):
 *   "mech_kernel"  5 (default) tile kernel, batch version 7: CTA per 4x4x4-box tile with
 *                  the halo staged in shared memory, trimmed candidate runs walked with a
 *                  conservative fp32 contact test (D32 <= min((r'_i+r'_j)^2, R^2(1+2^-12)),
 *                  the neighbour test for static candidates), one lane-parallel exact +
 *                  Eq. 4.1/4.2 pass over the survivors, ordered accumulation;
 *                  0 the same tiles with the version-6 batch (fp32 neighbour prefilter,
 *                  exact-test compaction, contact queue);
 *                  1 per-agent reference kernel reading neighbours from global memory;
 *                  2 the first tile kernel (per-lane pair lists, no run trimming);
 *                  3 version 6 with the packed f32x2 pair walk (4 CTAs per SM);
 *                  4 the row-broadcast kernel (2x4x8-box tiles, candidate words in
 *                  registers, agents broadcast, ballot masks; measured slower).
 *   "sir_index_capacity"  infected agents the SIR index holds (0 = max(65536, n/16)).
 *   "dense"        1 (default) / 0: regions too crowded for the tile kernel's shared-memory
 *                  staging (> 416 agents in a 6^3-box region) go to the dense-box kernel
 *                  (warp per box, broadcast candidate stream); 0: reference formulation.
 *   "diffuse_tma"  1 (default) / 0: bdm_diffuse streams the grid planes with TMA box loads
 *                  (nx even); 0, or nx odd: the register/shared-memory stencil kernel.
 *   "tile_depth"   0 (default) auto: two-tile work units when the first grid build of the
 *                  context had at most one agent per box, else one; 1 or 2 force it.
 *                  Two tiles stacked in z share one staged 6x6x10-box region, so sparse
 *                  populations fill the 32-lane batches (cfg5: -18 % k_mech).  3 (default
 *                  kernel only): two-tile units for denser populations, 8 warps sharing
 *                  a region of up to 672 staged agents, 3 CTAs per SM (same result; as
 *                  fast as depth 1 at cfg2, so never chosen automatically).
 *   "tile_order"   0 (default) row-major 4x4x4-box tiles; 1 blocked Hilbert: super-tiles
 *                  of 8^3 tiles row-major, the tiles inside one along a 3-D Hilbert
 *                  curve (the paper's Hilbert variant of agent
 *                  sorting).  Changes only the memory order of the sorted
 *                  agents; the slot array is re-sized at the next build.
 *   "sort_every"   K >= 0 (default 1): the mechanics step leaves the caller's arrays in
 *                  the grid's sorted order only on every K-th bdm_grid_build (counted
 *                  from this call; 0 = never) and otherwise writes every agent back
 *                  to its input index (the paper's sorting
 *                  frequency).  The state per id is identical for every K.
 *   "prefilter"    1 (default) / 0: conservative fp32 candidate test in the tile kernel
 *                  (never rejects a neighbour; the exact fp64 test decides).
 *   "fuse_reduce"  0 (default) / 1: bdm_mech_step also reduces the extent of the new
 *                  state (row a1 of the next step), and the next bdm_grid_build on the
 *                  same arrays (same x pointer and n) skips its own reduction.  The
 *                  caller must not modify positions or diameters in between (every
 *                  other bdm_* call that changes agents clears the fused extent).
 * All settings produce bit-identical results (per agent id; "tile_order" and
 * "sort_every" change only the memory order).  Errors: BDM_EINVAL for an unknown
 * name/value. */
bdm_status bdm_set_option(bdm_handle h, const char *name, int64_t value);

/* ---- Row f3: delta-encoded + LZ4-compressed aura messages ------------------------
 * Sec. "Data Transfer Minimization" (LZ4 evaluation P:6911-6937): sender
 * and receiver keep the same reference (a previous aura message); the sender reorders
 * the message to the reference, writes its difference against the reference and
 * compresses it; the receiver inverts both.  Readings R46-R51: the
 * reference is kept in ascending id order; slot r of the reference carries the message
 * agent with the same id (XOR of the IEEE bit patterns of x, y, z, d and of flags) or a
 * placeholder (presence bit 0); agents not in the reference follow in message order
 * (raw values + id); the payload is stored as byte planes and compressed as independent
 * 1024-byte LZ4 blocks (greedy parse, 11-bit hash).  Stream: 40-byte header (u32 magic
 * "BDA1", u32 1024, u64 nref, u64 nnew, u64 payload bytes, u32 chunks, u32 0), u32
 * compressed size per chunk, the chunks.  All arrays are device memory.  Ids must be
 * unique within a message.  Messages of up to 2^31 - 1 agents. */

/* Upper bound of the stream size for a reference of nref agents and a message of n
 * agents (host-only; -1 for negative sizes). */
int64_t bdm_aura_max_size(int64_t nref, int64_t n);

/* ref := msg sorted by ascending id (R46; hand-written LSD radix sort of (id, index) pairs, four 8-bit passes, + gather).  ref->capacity >=
 * msg->n; sets ref->n.  Asynchronous on `stream`.  Errors: BDM_EINVAL (NULL arrays),
 * BDM_ECAPACITY. */
bdm_status bdm_aura_reference(bdm_handle h, const bdm_agents *msg, bdm_agents *ref, void *stream);

/* Encodes msg against ref (R47-R50) into the device buffer out (out_cap bytes).
 * Synchronizing; *out_size_host = stream bytes.  msg is not modified.  Errors:
 * BDM_ECAPACITY if out_cap is too small (nothing meaningful is written; *out_size_host
 * holds the size needed), BDM_EINVAL for NULL arguments. */
bdm_status bdm_aura_encode(bdm_handle h, const bdm_agents *msg, const bdm_agents *ref,
                           uint8_t *out, int64_t out_cap, int64_t *out_size_host, void *stream);

/* Decodes the device stream in[0, in_size) against ref (the receiver's copy of the
 * sender's reference) into msg (R51: the reference-order survivors, then the new
 * agents); sets msg->n.  Synchronizing.  Errors: BDM_EINVAL for a malformed stream or
 * one encoded against a reference of another size, BDM_ECAPACITY if msg->capacity is
 * too small (msg unchanged). */
bdm_status bdm_aura_decode(bdm_handle h, const uint8_t *in, int64_t in_size, const bdm_agents *ref,
                           bdm_agents *msg, void *stream);

/* Host-only query of the tile numbering inside an 8^3 super-tile (option "tile_order"):
 * rank_out[x | y<<3 | z<<6] = position of local tile (x, y, z) along the curve, for
 * order 0 (row-major, the identity) or 1 (3-D Hilbert curve, Skilling's transform).
 * rank_out: caller-owned host array of 512 entries.  No GPU needed.
 * Errors: BDM_EINVAL for NULL or a bad order. */
bdm_status bdm_tile_curve(int32_t order, uint16_t *rank_out);

/* Diagnostic: measured fp64 FMA throughput of this GPU (DFMA lane-operations per
 * second, i.e. half the fp64 FLOP/s) and the SM count.  Synchronizing. */
bdm_status bdm_peak_dfma(bdm_handle h, double *dfma_per_s, int32_t *sm_count);

/* Diagnostic: checks the SIR step's shared-reciprocal quotient (kernels_sir.cu,
 * div_by_recip: three IEEE divisions v/|v| of Alg. 9's capped step, from
 * one reciprocal) against the hardware's IEEE division on n seeded random operands of
 * the step's range (v = 2u - 1 per axis with u = w 2^-32, |v| > 1) and counts the
 * results that differ in any bit.  mismatches: caller-owned host pointer.
 * Synchronizing.  Errors: BDM_EINVAL for NULL or n <= 0. */
bdm_status bdm_selftest_recip_div(bdm_handle h, int64_t n, uint64_t seed,
                                  unsigned long long *mismatches);

#ifdef __cplusplus
}
#endif
#endif /* BDM_H */
