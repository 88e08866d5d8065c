// bdm_abi.cu -- extern "C" entry points of include/bdm.h: argument checks, workspace
// management, and the stream-ordered composition of the kernels.
#include <cuda_runtime.h>
#include <stdio.h>
#include <math.h>
#include <string.h>

#include <string>

#include "bdm_internal.cuh"

namespace bdm {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

bdm_status cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return BDM_ECUDA;
}

int64_t scan_block_count(int64_t slot_cap);

static bdm_status fail(bdm_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

template <class T>
static bdm_status dalloc(Ctx *c, T **p, int64_t count) {
    if (*p) ctx_free(c, *p);
    *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = ctx_malloc(c, (void **)p, (size_t)count * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return fail(BDM_ECAPACITY, std::string("allocation of ") +
                                       std::to_string((long long)count * sizeof(T)) +
                                       " bytes failed: " + cudaGetErrorString(e));
    }
    return BDM_OK;
}

static bdm_status grow_agents(Ctx *c, int64_t n) {
    if (n <= c->agent_cap) return BDM_OK;
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    // exact on the first sizing (the caller's stated maximum), with slack on regrowth
    const int64_t cap = c->agent_cap == 0 ? n : n + n / 8 + 1024;
    // optional buffers are re-allocated at the new size on their next use
    void *opt[] = {c->svol, c->div_rank, c->lrank, c->cls, c->cls2, c->perm};
    for (void *p : opt)
        if (p) ctx_free(c, p);
    c->svol = nullptr;
    c->div_rank = c->lrank = c->cls = c->cls2 = c->perm = nullptr;
    bdm_status s;
    if ((s = dalloc(c, &c->key, cap)) || (s = dalloc(c, &c->rank, cap)) ||
        (s = dalloc(c, &c->perm_tmp, cap)) || (s = dalloc(c, &c->skey, cap)) ||
        (s = dalloc(c, &c->sid, cap)) || (s = dalloc(c, &c->sx, cap)) ||
        (s = dalloc(c, &c->sy, cap)) || (s = dalloc(c, &c->sz, cap)) || (s = dalloc(c, &c->sd, cap)) ||
        (s = dalloc(c, &c->sidf, cap)) || (s = dalloc(c, &c->sflags, cap))) {
        c->agent_cap = 0;
        return s;
    }
    c->agent_cap = cap;
    c->grid_valid = false;
    // the scan block sums serve both the slot scan and the agent-indexed scans
    const int64_t nb = scan_block_count(cap > c->slot_cap ? cap : c->slot_cap) + 1;
    if (nb > c->block_sums_cap) {
        if ((s = dalloc(c, &c->block_sums, nb))) return s;
        c->block_sums_cap = nb;
    }
    return BDM_OK;
}

static bdm_status grow_slots(Ctx *c, int64_t nslots) {
    if (nslots <= c->slot_cap) return BDM_OK;
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    bdm_status s;
    if ((s = dalloc(c, &c->box_start, nslots + 1)) || (s = dalloc(c, &c->dense_list, 2 * (nslots / 64) + 2))) {
        c->slot_cap = 0;
        return s;
    }
    const int64_t nb = scan_block_count(nslots > c->agent_cap ? nslots : c->agent_cap) + 1;
    if (nb > c->block_sums_cap) {
        if ((s = dalloc(c, &c->block_sums, nb))) { c->slot_cap = 0; return s; }
        c->block_sums_cap = nb;
    }
    c->slot_cap = nslots;
    long long cap = nslots;
    BDM_CUDA_TRY(cudaMemcpy(&c->sc->slot_cap, &cap, sizeof(cap), cudaMemcpyHostToDevice));
    c->grid_valid = false;
    return BDM_OK;
}

static bdm_status check_agents(const bdm_agents *a, bool need_all) {
    if (!a) return fail(BDM_EINVAL, "agents is NULL");
    if (a->n < 0 || a->n > a->capacity) return fail(BDM_EINVAL, "n < 0 or n > capacity");
    if (a->n > 0xFFFFFFFFll - 1) return fail(BDM_EINVAL, "n exceeds 2^32 - 2 agents per context");
    if (need_all && a->n > 0 &&
        (!a->x || !a->y || !a->z || !a->diameter || !a->id || !a->flags))
        return fail(BDM_EINVAL, "a required agent array is NULL");
    const void *ptrs[] = {a->x, a->y, a->z, a->diameter, a->volume};
    for (const void *p : ptrs)
        if (((uintptr_t)p & 7u) != 0) return fail(BDM_EINVAL, "agent array not 8-byte aligned");
    return BDM_OK;
}

// Latched device conditions -> status (after a synchronize).
static bdm_status read_latches(Ctx *c, bool clear) {
    BDM_CUDA_TRY(cudaMemcpy(c->sc_host, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost));
    bdm_status st = BDM_OK;
    if (c->sc_host->nonfinite) {
        st = fail(BDM_ENOTFINITE, "a position or diameter is NaN/Inf");
    } else if (c->sc_host->overflow == 6) {
        st = fail(BDM_EINVAL, "toroidal boundary needs at least 3 boxes of edge >= R per axis "
                              "(side >= 3 R)");
    } else if (c->sc_host->overflow == 5) {
        st = fail(BDM_EINVAL, "growth/division needs ids exactly 0..n-1 (an id is >= n)");
    } else if (c->sc_host->overflow == 4) {
        st = fail(BDM_ECAPACITY, "slab send buffer too small");
    } else if (c->sc_host->overflow == 3) {
        st = fail(BDM_ECAPACITY, "SIR infected index too small (raise option sir_index_capacity)");
    } else if (c->sc_host->overflow == 2) {
        st = fail(BDM_ECAPACITY, "agent capacity too small for the daughters of this step");
    } else if (c->sc_host->overflow) {
        st = fail(BDM_ECAPACITY, "grid needs " + std::to_string(c->sc_host->nslots) +
                                     " slots, capacity " + std::to_string(c->slot_cap));
    }
    if (st != BDM_OK) c->fused_valid = false;  // a skipped step leaves no fused extent
    if (clear && st != BDM_OK) {
        int32_t z[2] = {0, 0};
        BDM_CUDA_TRY(cudaMemcpy(&c->sc->overflow, z, sizeof(z), cudaMemcpyHostToDevice));
    }
    return st;
}

// Skilling's transform (AxesToTranspose, "Programming the Hilbert curve", 2004) of
// the b-bit coordinates X[0..n) into the transposed Hilbert index.
static void axes_to_transpose(uint32_t *X, int b, int n) {
    const uint32_t M = 1u << (b - 1);
    for (uint32_t Q = M; Q > 1; Q >>= 1) {  // inverse undo
        const uint32_t P = Q - 1;
        for (int i = 0; i < n; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    for (int i = 1; i < n; ++i) X[i] ^= X[i - 1];  // Gray encode
    uint32_t t = 0;
    for (uint32_t Q = M; Q > 1; Q >>= 1)
        if (X[n - 1] & Q) t ^= Q - 1;
    for (int i = 0; i < n; ++i) X[i] ^= t;
}

// Curve position of each tile (x | y<<3 | z<<6) of an 8^3 super-tile.
static void tile_curve(int order, uint16_t *rank, uint16_t *inv) {
    for (uint32_t l = 0; l < 512; ++l) {
        uint32_t r = l;
        if (order == 1) {
            uint32_t X[3] = {l & 7u, (l >> 3) & 7u, l >> 6};
            axes_to_transpose(X, 3, 3);
            r = 0;
            for (int b = 2; b >= 0; --b)
                for (int i = 0; i < 3; ++i) r = (r << 1) | ((X[i] >> b) & 1u);
        }
        rank[l] = (uint16_t)r;
        if (inv) inv[r] = (uint16_t)l;
    }
}

// Makes the context's device current for one entry point and restores the caller's
// (contexts on several devices may share a thread).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(bdm_handle h) {
        if (!h) return;
        const int want = ((Ctx *)h)->device;
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != want) cudaSetDevice(want);
        else prev = -1;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace bdm

using namespace bdm;

extern "C" {

const char *bdm_last_error(void) { return g_err.c_str(); }

const char *bdm_version(void) { return "bdm 0.1.0 sm_100a"; }

bdm_status bdm_create(bdm_handle *out, int device, int64_t max_agents) {
    return bdm_create_ex(out, device, max_agents, 0, nullptr, nullptr, nullptr);
}

bdm_status bdm_create_ex(bdm_handle *out, int device, int64_t max_agents, int64_t max_ghosts,
                         bdm_alloc_fn alloc, bdm_free_fn release, void *user) {
    if (!out) return fail(BDM_EINVAL, "out is NULL");
    *out = nullptr;
    if (max_agents < 0 || max_ghosts < 0) return fail(BDM_EINVAL, "max_agents < 0 or max_ghosts < 0");
    if ((alloc == nullptr) != (release == nullptr))
        return fail(BDM_EINVAL, "alloc and release must both be given or both be NULL");
    if (max_agents + max_ghosts > 0xFFFFFFFFll - 1)
        return fail(BDM_EINVAL, "max_agents + max_ghosts exceeds 2^32 - 2 agents per context");
    int ndev = 0;
    BDM_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev || device >= kMaxDevices)
        return fail(BDM_EINVAL, "bad device index");
    BDM_CUDA_TRY(cudaSetDevice(device));
    Ctx *c = new Ctx();
    c->device = device;
    c->alloc_fn = alloc;
    c->free_fn = release;
    c->alloc_ctx = user;
    c->max_ghosts = max_ghosts;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaMalloc(&c->sc, sizeof(DevScalars)) != cudaSuccess ||
        cudaMallocHost(&c->sc_host, sizeof(DevScalars)) != cudaSuccess ||
        cudaMallocHost(&c->dims_hint, 4 * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&c->pair_count, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->n_new, sizeof(long long)) != cudaSuccess ||
        cudaMalloc(&c->pack_counts, 16 * sizeof(long long)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return fail(BDM_ECUDA, "allocation of the context scalars failed");
    }
    cudaMemset(c->sc, 0, sizeof(DevScalars));
    c->dims_hint[0] = c->dims_hint[1] = c->dims_hint[2] = 0;
    bdm_status s = grow_agents(c, max_agents + max_ghosts > 0 ? max_agents + max_ghosts : 1);
    if (s != BDM_OK) {
        bdm_destroy((bdm_handle)c);
        return s;
    }
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    *out = (bdm_handle)c;
    return BDM_OK;
}

bdm_status bdm_destroy(bdm_handle h) {
    if (!h) return BDM_OK;
    Ctx *c = (Ctx *)h;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    free_aura(c);
    free_dist(c);
    void *bufs[] = {c->key, c->rank, c->perm_tmp, c->skey, c->sid, c->perm, c->sx, c->sy,
                    c->sz, c->sd, c->sidf, c->sflags, c->svol, c->div_rank, c->box_start, c->dense_list, c->dense_scr,
                    c->onco_id, c->onco_out,
                    c->block_sums, c->scan_state, c->pair_count, c->n_new, c->lrank, c->cls, c->cls2,
                    c->pack_counts, c->sc};
    for (void *p : bufs)
        if (p) ctx_free(c, p);
    void *sbufs[] = {c->sir.keys, c->sir.heads, c->sir.next, c->sir.bitmap, c->sir.ix, c->sir.iy,
                     c->sir.iz, c->sir.misc};
    for (void *q : sbufs)
        if (q) cudaFree(q);
    if (c->sc_host) cudaFreeHost(c->sc_host);
    if (c->dims_hint) cudaFreeHost(c->dims_hint);
    if (c->hint_ev) cudaEventDestroy(c->hint_ev);
    delete c;
    return BDM_OK;
}

bdm_status bdm_init_spheres(bdm_handle h, bdm_agents *a, int64_t id0, int64_t n, uint64_t seed,
                            double side, double d_lo, double d_width, int32_t d_random,
                            void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    if (!a || n < 0 || n > a->capacity || id0 < 0)
        return fail(BDM_EINVAL, "bad n / id0 / capacity");
    if (n > 0 && (!a->x || !a->y || !a->z || !a->diameter || !a->id || !a->flags))
        return fail(BDM_EINVAL, "a required agent array is NULL");
    if (!(side > 0.0)) return fail(BDM_EINVAL, "side must be > 0");
    a->n = n;
    return launch_init_spheres(a, id0, n, seed, side, d_lo, d_width, d_random,
                               (cudaStream_t)stream);
}

bdm_status bdm_grid_build(bdm_handle h, const bdm_agents *a, const bdm_agents *ghosts,
                          double radius, void *stream) {
    DeviceScope ds__(h);
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    Ctx *c = (Ctx *)h;
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    if (ghosts && ghosts->n > 0 && (s = check_agents(ghosts, true)) != BDM_OK) return s;
    const bdm_agents *g = (ghosts && ghosts->n > 0) ? ghosts : nullptr;
    if (radius < 0.0 || radius != radius) return fail(BDM_EINVAL, "radius < 0");
    cudaStream_t st = (cudaStream_t)stream;
    c->grid_valid = false;
    const int64_t ntot = a->n + (g ? g->n : 0);
    if (a->n == 0) {
        c->grid_valid = true;
        c->grid_x = a->x;
        c->grid_n = 0;
        c->grid_ng = 0;
        return BDM_OK;
    }
    if ((s = grow_agents(c, ntot)) != BDM_OK) return s;
    if ((s = launch_grid_geometry(c, a, g, radius, st)) != BDM_OK) return s;
    if (c->slot_cap == 0) {
        // first build: size the slot array from the actual geometry (one sync),
        // with room for growth of the open-boundary space (+4 tiles per axis)
        BDM_CUDA_TRY(cudaStreamSynchronize(st));
        BDM_CUDA_TRY(cudaMemcpy(c->sc_host, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost));
        if (c->sc_host->nonfinite) {
            int32_t z[2] = {0, 0};
            cudaMemcpy(&c->sc->overflow, z, sizeof(z), cudaMemcpyHostToDevice);
            return fail(BDM_ENOTFINITE, "a position or diameter is NaN/Inf");
        }
        // (+8 in blocked Hilbert order: T is padded to whole super-tiles)
        c->density_hint = (double)ntot / ((double)c->sc_host->dims[0] * (double)c->sc_host->dims[1] *
                                          (double)c->sc_host->dims[2]);
        const int64_t pad = c->tile_order ? 8 : 4;
        const int64_t t0 = c->sc_host->T[0] + pad, t1 = c->sc_host->T[1] + pad,
                      t2 = c->sc_host->T[2] + pad;
        if ((s = grow_slots(c, t0 * t1 * t2 * 64)) != BDM_OK) return s;
        int32_t z[2] = {0, 0};
        BDM_CUDA_TRY(cudaMemcpy(&c->sc->overflow, z, sizeof(z), cudaMemcpyHostToDevice));
        if ((s = launch_grid_geometry(c, a, g, radius, st)) != BDM_OK) return s;
    }
    if ((s = launch_grid_sort(c, a, g, st)) != BDM_OK) return s;
    // every 8th build the box counts travel to a pinned mirror in stream order; later
    // mechanics launches read whatever has arrived as their auto tile-depth hint (no
    // synchronization; the hint only picks the faster of two exact kernels)
    // (the host reads the mirror only after the event recorded behind the copy has
    // completed, together with the agent count saved with it)
    if (c->tile_depth == 0 && (c->grid_builds & 7) == 1 && !c->hint_pending) {
        if (!c->hint_ev) BDM_CUDA_TRY(cudaEventCreateWithFlags(&c->hint_ev, cudaEventDisableTiming));
        BDM_CUDA_TRY(cudaMemcpyAsync(c->dims_hint, c->sc->dims, sizeof(c->sc->dims),
                                     cudaMemcpyDeviceToHost, st));
        BDM_CUDA_TRY(cudaEventRecord(c->hint_ev, st));
        c->hint_n = ntot;
        c->hint_pending = true;
    }
    c->grid_valid = true;
    c->grid_x = a->x;
    c->grid_n = a->n;
    c->grid_ng = g ? g->n : 0;
    c->grid_torus = c->torus_side;
    return BDM_OK;
}

bdm_status bdm_mech_step(bdm_handle h, bdm_agents *a, const bdm_params *p, void *stream) {
    DeviceScope ds__(h);
    if (!h || !p) return fail(BDM_EINVAL, "handle or params is NULL");
    Ctx *c = (Ctx *)h;
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    if (!c->grid_valid || c->grid_x != a->x || c->grid_n != a->n)
        return fail(BDM_EINVAL, "bdm_mech_step needs a preceding bdm_grid_build on the same agents");
    if (p->boundary != 0 && p->boundary != 1 && p->boundary != 2) return fail(BDM_EINVAL, "bad boundary");
    if ((p->boundary == 2) != (c->grid_torus > 0.0) || (p->boundary == 2 && c->grid_torus != p->hi[0]))
        return fail(BDM_EINVAL, "toroidal mechanics needs the grid built on the same torus (bdm_step)");
    if (!(p->dt >= 0.0) || !(p->max_displacement >= 0.0) || !(p->force_threshold >= 0.0))
        return fail(BDM_EINVAL, "dt, max_displacement and force_threshold must be >= 0");
    c->grid_valid = false;  // positions change: the grid is stale afterwards
    if (a->n == 0) return BDM_OK;
    // the kernels sweep locals + ghosts of the build; outputs go to the locals only
    bdm_agents all = *a;
    all.n = a->n + c->grid_ng;
    const bdm_status s2 = launch_mech(c, &all, p, (cudaStream_t)stream);
    c->fused_valid = (s2 == BDM_OK) && c->fuse_reduce && c->grid_ng == 0;
    c->fused_x = a->x;
    c->fused_n = a->n;
    return s2;
}

bdm_status bdm_step(bdm_handle h, bdm_agents *a, const bdm_params *p, void *stream) {
    DeviceScope ds__(h);
    if (!p || !h) return fail(BDM_EINVAL, "handle or params is NULL");
    Ctx *c = (Ctx *)h;
    if (p->boundary == 2) {  // toroidal (R52): the cube [0, hi[0])^3
        const double L = p->hi[0];
        if (!(L > 0.0) || p->hi[1] != L || p->hi[2] != L || p->lo[0] != 0.0 || p->lo[1] != 0.0 ||
            p->lo[2] != 0.0)
            return fail(BDM_EINVAL, "toroidal boundary needs lo = 0 and a cube hi[0] = hi[1] = hi[2] > 0");
        c->torus_side = L;
    }
    bdm_status s = bdm_grid_build(h, a, nullptr, p->radius, stream);
    c->torus_side = 0.0;
    if (s != BDM_OK) return s;
    return bdm_mech_step(h, a, p, stream);
}

bdm_status bdm_step_host(bdm_handle h, const bdm_agents *hin, bdm_agents *hout, bdm_agents *dev,
                         const bdm_params *p, void *stream) {
    DeviceScope ds__(h);
    if (!h || !hin || !hout || !dev || !p) return fail(BDM_EINVAL, "NULL argument");
    if (hin->n > dev->capacity || hin->n > hout->capacity)
        return fail(BDM_EINVAL, "n exceeds a capacity");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)hin->n;
    dev->n = hin->n;
    ((Ctx *)h)->fused_valid = false;  // the device arrays are overwritten from the host
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->x, hin->x, n * 8, cudaMemcpyHostToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->y, hin->y, n * 8, cudaMemcpyHostToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->z, hin->z, n * 8, cudaMemcpyHostToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->diameter, hin->diameter, n * 8, cudaMemcpyHostToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->id, hin->id, n * 4, cudaMemcpyHostToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dev->flags, hin->flags, n * 4, cudaMemcpyHostToDevice, st));
    bdm_status s = bdm_step(h, dev, p, stream);
    if (s != BDM_OK) return s;
    hout->n = hin->n;
    BDM_CUDA_TRY(cudaMemcpyAsync(hout->x, dev->x, n * 8, cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(hout->y, dev->y, n * 8, cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(hout->z, dev->z, n * 8, cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(hout->flags, dev->flags, n * 4, cudaMemcpyDeviceToHost, st));
    // a step that kept the input order (option sort_every) leaves d and id where they
    // were: in place they are already on the host
    const bool inplace = hout->diameter == hin->diameter && hout->id == hin->id;
    if (!(inplace && ((Ctx *)h)->keep_order)) {
        BDM_CUDA_TRY(cudaMemcpyAsync(hout->diameter, dev->diameter, n * 8, cudaMemcpyDeviceToHost, st));
        BDM_CUDA_TRY(cudaMemcpyAsync(hout->id, dev->id, n * 4, cudaMemcpyDeviceToHost, st));
    }
    return bdm_sync(h, stream);
}

// K end-to-end steps on a host state, pipelined: the device -> host copy of step k's
// result and the host -> device copy of step k+1's input run concurrently, chunk by
// chunk (chunk c of step k+1 goes up as soon as chunk c of step k has come down), on
// two copy streams next to the compute stream -- PCIe is full duplex.
bdm_status bdm_run_host(bdm_handle h, bdm_agents *host, bdm_agents *dev, const bdm_params *p,
                        int32_t steps, int32_t chunks, void *stream) {
    DeviceScope ds__(h);
    if (!h || !host || !dev || !p) return fail(BDM_EINVAL, "NULL argument");
    if (steps < 0 || chunks < 1 || chunks > 64) return fail(BDM_EINVAL, "steps < 0 or chunks not in 1..64");
    if (host->n > dev->capacity) return fail(BDM_EINVAL, "n exceeds the device capacity");
    Ctx *c = (Ctx *)h;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = host->n;
    dev->n = n;
    if (steps == 0 || n == 0) return BDM_OK;
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ev_up = nullptr, ev_comp = nullptr, ev_down[64] = {};
    bdm_status res = BDM_OK;
    auto cleanup = [&]() {
        if (up) cudaStreamSynchronize(up);
        if (down) cudaStreamSynchronize(down);
        for (int k = 0; k < chunks; ++k)
            if (ev_down[k]) cudaEventDestroy(ev_down[k]);
        if (ev_up) cudaEventDestroy(ev_up);
        if (ev_comp) cudaEventDestroy(ev_comp);
        if (up) cudaStreamDestroy(up);
        if (down) cudaStreamDestroy(down);
    };
#define BDM_RH_TRY(expr)                                              \
    do {                                                              \
        cudaError_t e__ = (expr);                                     \
        if (e__ != cudaSuccess) {                                     \
            res = cuda_fail(e__, #expr);                              \
            cleanup();                                                \
            return res;                                               \
        }                                                             \
    } while (0)
    BDM_RH_TRY(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    BDM_RH_TRY(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
    BDM_RH_TRY(cudaEventCreateWithFlags(&ev_up, cudaEventDisableTiming));
    BDM_RH_TRY(cudaEventCreateWithFlags(&ev_comp, cudaEventDisableTiming));
    for (int k = 0; k < chunks; ++k) BDM_RH_TRY(cudaEventCreateWithFlags(&ev_down[k], cudaEventDisableTiming));
    // the compute stream's earlier work (the caller's) precedes the first upload
    BDM_RH_TRY(cudaEventRecord(ev_comp, st));
    BDM_RH_TRY(cudaStreamWaitEvent(up, ev_comp, 0));
    for (int32_t t = 0; t < steps; ++t) {
        for (int k = 0; k < chunks; ++k) {
            const int64_t a = n * k / chunks, b = n * (k + 1) / chunks;
            if (b == a) continue;
            const size_t m = (size_t)(b - a);
            if (t > 0) BDM_RH_TRY(cudaStreamWaitEvent(up, ev_down[k], 0));
            BDM_RH_TRY(cudaMemcpyAsync(dev->x + a, host->x + a, m * 8, cudaMemcpyHostToDevice, up));
            BDM_RH_TRY(cudaMemcpyAsync(dev->y + a, host->y + a, m * 8, cudaMemcpyHostToDevice, up));
            BDM_RH_TRY(cudaMemcpyAsync(dev->z + a, host->z + a, m * 8, cudaMemcpyHostToDevice, up));
            BDM_RH_TRY(cudaMemcpyAsync(dev->diameter + a, host->diameter + a, m * 8, cudaMemcpyHostToDevice, up));
            BDM_RH_TRY(cudaMemcpyAsync(dev->id + a, host->id + a, m * 4, cudaMemcpyHostToDevice, up));
            BDM_RH_TRY(cudaMemcpyAsync(dev->flags + a, host->flags + a, m * 4, cudaMemcpyHostToDevice, up));
        }
        BDM_RH_TRY(cudaEventRecord(ev_up, up));
        BDM_RH_TRY(cudaStreamWaitEvent(st, ev_up, 0));
        c->fused_valid = false;  // the device arrays were overwritten from the host
        const bdm_status s = bdm_step(h, dev, p, stream);
        if (s != BDM_OK) {
            cleanup();
            return s;
        }
        // a step that kept the input order (option sort_every) leaves d and id in place
        const bool all = !c->keep_order;
        BDM_RH_TRY(cudaEventRecord(ev_comp, st));
        BDM_RH_TRY(cudaStreamWaitEvent(down, ev_comp, 0));
        for (int k = 0; k < chunks; ++k) {
            const int64_t a = n * k / chunks, b = n * (k + 1) / chunks;
            const size_t m = (size_t)(b - a);
            if (m) {
                BDM_RH_TRY(cudaMemcpyAsync(host->x + a, dev->x + a, m * 8, cudaMemcpyDeviceToHost, down));
                BDM_RH_TRY(cudaMemcpyAsync(host->y + a, dev->y + a, m * 8, cudaMemcpyDeviceToHost, down));
                BDM_RH_TRY(cudaMemcpyAsync(host->z + a, dev->z + a, m * 8, cudaMemcpyDeviceToHost, down));
                BDM_RH_TRY(cudaMemcpyAsync(host->flags + a, dev->flags + a, m * 4, cudaMemcpyDeviceToHost, down));
                if (all) {
                    BDM_RH_TRY(cudaMemcpyAsync(host->diameter + a, dev->diameter + a, m * 8,
                                               cudaMemcpyDeviceToHost, down));
                    BDM_RH_TRY(cudaMemcpyAsync(host->id + a, dev->id + a, m * 4, cudaMemcpyDeviceToHost, down));
                }
            }
            BDM_RH_TRY(cudaEventRecord(ev_down[k], down));
        }
    }
    // the caller's stream resumes after the last download
    BDM_RH_TRY(cudaEventRecord(ev_comp, down));
    BDM_RH_TRY(cudaStreamWaitEvent(st, ev_comp, 0));
#undef BDM_RH_TRY
    cleanup();
    return bdm_sync(h, stream);
}

bdm_status bdm_grow_divide(bdm_handle h, bdm_agents *a, const bdm_params *p, double growth,
                           double v_max, int64_t *n_out_host, void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !p || !n_out_host) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    if (!a->volume) return fail(BDM_EINVAL, "growth/division needs the volume array");
    if (!(growth >= 0.0) || !(v_max > 0.0)) return fail(BDM_EINVAL, "growth < 0 or v_max <= 0");
    if ((s = grow_agents(c, a->n)) != BDM_OK) return s;
    c->grid_valid = false;
    const double vol_to_r3 = 0.75 / M_PI;  // r^3 = V * 0.75/pi, computed once (R28)
    return launch_grow_divide(c, a, growth, v_max, vol_to_r3, p->seed, p->step,
                              (long long *)n_out_host, (cudaStream_t)stream);
}

bdm_status bdm_onco_step(bdm_handle h, bdm_agents *a, uint32_t *age, int64_t age_cap,
                         const bdm_onco_params *p, int64_t id_next, int64_t *out_host,
                         void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !p || !out_host) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    if (a->n > 0 && (!a->volume || !age)) return fail(BDM_EINVAL, "oncology needs volume and age");
    if (id_next < a->n || id_next > 0xFFFFFFFFll)
        return fail(BDM_EINVAL, "id_next must be >= n (ids < id_next) and < 2^32");
    if (age_cap < id_next) return fail(BDM_EINVAL, "age_cap < id_next");
    if (!(p->growth >= 0.0) || !(p->max_diameter >= 0.0) || !(p->p_death >= 0.0) ||
        !(p->p_div >= 0.0))
        return fail(BDM_EINVAL, "negative oncology parameter");
    if ((s = grow_agents(c, a->capacity)) != BDM_OK) return s;
    const int64_t nb = scan_block_count(id_next + 1) + 1;
    if (nb > c->block_sums_cap) {
        BDM_CUDA_TRY(cudaDeviceSynchronize());
        if ((s = dalloc(c, &c->block_sums, nb)) != BDM_OK) return s;
        c->block_sums_cap = nb;
    }
    c->grid_valid = false;
    return launch_onco_step(c, a, age, age_cap, p, id_next, (long long *)out_host,
                            (cudaStream_t)stream);
}

bdm_status bdm_sir_step(bdm_handle h, bdm_agents *a, const bdm_params *p, double side,
                        double radius, double p_inf, double p_rec, int64_t *counts_host,
                        void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !p || !a) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    if (a->n < 0 || a->n > a->capacity) return fail(BDM_EINVAL, "n < 0 or n > capacity");
    if (a->n > 0 && (!a->x || !a->y || !a->z || !a->state))
        return fail(BDM_EINVAL, "SIR needs x, y, z and state");
    if (!(side > 0.0) || !(radius > 0.0)) return fail(BDM_EINVAL, "side and radius must be > 0");
    if (!(p_inf >= 0.0 && p_inf <= 1.0) || !(p_rec >= 0.0 && p_rec <= 1.0))
        return fail(BDM_EINVAL, "probabilities must be in [0, 1]");
    c->grid_valid = false;
    return launch_sir_step(c, a, p, side, radius, p_inf, p_rec, (long long *)counts_host,
                           (cudaStream_t)stream);
}

static bdm_status check_grid3(const bdm_grid3 *g) {
    if (!g) return fail(BDM_EINVAL, "grid is NULL");
    if (g->nx < 0 || g->ny < 0 || g->nz < 0) return fail(BDM_EINVAL, "negative grid size");
    if (g->nx * g->ny >= (1ll << 31) || g->nz >= (1ll << 31))
        return fail(BDM_EINVAL, "grid too large (nx*ny and nz must be < 2^31)");
    if (!(g->dx > 0.0) || !(g->dy > 0.0) || !(g->dz > 0.0))
        return fail(BDM_EINVAL, "grid spacing must be > 0");
    return BDM_OK;
}

bdm_status bdm_diffuse(bdm_handle h, const double *u_in, double *u_out, const bdm_grid3 *g,
                       double nu, double mu, double dt, void *stream) {
    DeviceScope ds__(h);
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    bdm_status s = check_grid3(g);
    if (s != BDM_OK) return s;
    if (g->nx * g->ny * g->nz > 0 && (!u_in || !u_out || u_in == u_out))
        return fail(BDM_EINVAL, "u_in and u_out must be distinct device buffers");
    return launch_diffuse((Ctx *)h, u_in, u_out, g, nu, mu, dt, (cudaStream_t)stream);
}

bdm_status bdm_secrete(bdm_handle h, const bdm_agents *a, const uint8_t *type, int32_t type_sel,
                       double q, double *u, const bdm_grid3 *g, void *stream) {
    DeviceScope ds__(h);
    if (!h || !a) return fail(BDM_EINVAL, "NULL argument");
    bdm_status s = check_grid3(g);
    if (s != BDM_OK) return s;
    if (a->n < 0 || a->n > a->capacity) return fail(BDM_EINVAL, "n < 0 or n > capacity");
    if (a->n > 0 && (!a->x || !a->y || !a->z || !type || !u))
        return fail(BDM_EINVAL, "secretion needs x, y, z, type and the grid");
    if (g->nx * g->ny * g->nz == 0 && a->n > 0) return fail(BDM_EINVAL, "empty grid");
    return launch_secrete((Ctx *)h, a, type, type_sel, q, u, g, (cudaStream_t)stream);
}

bdm_status bdm_chemotaxis(bdm_handle h, bdm_agents *a, const uint8_t *type, int32_t type_sel,
                          double weight, const double *u, const bdm_grid3 *g, void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !a) return fail(BDM_EINVAL, "NULL argument");
    bdm_status s = check_grid3(g);
    if (s != BDM_OK) return s;
    if (a->n < 0 || a->n > a->capacity) return fail(BDM_EINVAL, "n < 0 or n > capacity");
    if (a->n > 0 && (!a->x || !a->y || !a->z || !type || !u))
        return fail(BDM_EINVAL, "chemotaxis needs x, y, z, type and the grid");
    if (g->nx * g->ny * g->nz == 0 && a->n > 0) return fail(BDM_EINVAL, "empty grid");
    ((Ctx *)h)->grid_valid = false;
    return launch_chemotaxis((Ctx *)h, a, type, type_sel, weight, u, g, (cudaStream_t)stream);
}

bdm_status bdm_local_frame(bdm_handle h, const bdm_agents *a, double *frame_dev, void *stream) {
    DeviceScope ds__(h);
    if (!h || !a || !frame_dev) return fail(BDM_EINVAL, "NULL argument");
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    return launch_local_frame((Ctx *)h, a, frame_dev, (cudaStream_t)stream);
}

bdm_status bdm_set_frame(bdm_handle h, const double *frame_dev) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    Ctx *c = (Ctx *)h;
    c->frame = frame_dev;
    c->grid_valid = false;
    return BDM_OK;
}

bdm_status bdm_pack_slab(bdm_handle h, bdm_agents *a, double lo, double hi, double margin,
                         int32_t what, bdm_agents *to_left, bdm_agents *to_right,
                         int64_t *counts_host, void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !a || !to_left || !to_right || !counts_host) return fail(BDM_EINVAL, "NULL argument");
    if (what != BDM_PACK_MIGRATE && what != BDM_PACK_AURA) return fail(BDM_EINVAL, "bad what");
    if (!(lo <= hi) || !(margin >= 0.0)) return fail(BDM_EINVAL, "need lo <= hi and margin >= 0");
    Ctx *c = (Ctx *)h;
    bdm_status s = check_agents(a, true);
    if (s != BDM_OK) return s;
    if ((s = grow_agents(c, a->n)) != BDM_OK) return s;
    c->grid_valid = false;  // the migration compaction uses the sorted workspace
    return launch_pack_slab(c, a, lo, hi, margin, what, to_left, to_right,
                            (long long *)counts_host, (cudaStream_t)stream);
}

bdm_status bdm_append(bdm_handle h, bdm_agents *dst, const bdm_agents *src, void *stream) {
    DeviceScope ds__(h);
    if (h) ((Ctx *)h)->fused_valid = false;
    if (!h || !dst || !src) return fail(BDM_EINVAL, "NULL argument");
    if (src->n < 0 || dst->n < 0) return fail(BDM_EINVAL, "negative n");
    if (dst->n + src->n > dst->capacity) return fail(BDM_ECAPACITY, "append exceeds capacity");
    if (src->n == 0) return BDM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)src->n, o = (size_t)dst->n;
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->x + o, src->x, n * 8, cudaMemcpyDeviceToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->y + o, src->y, n * 8, cudaMemcpyDeviceToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->z + o, src->z, n * 8, cudaMemcpyDeviceToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->diameter + o, src->diameter, n * 8, cudaMemcpyDeviceToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->id + o, src->id, n * 4, cudaMemcpyDeviceToDevice, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(dst->flags + o, src->flags, n * 4, cudaMemcpyDeviceToDevice, st));
    if (dst->volume && src->volume)
        BDM_CUDA_TRY(cudaMemcpyAsync(dst->volume + o, src->volume, n * 8, cudaMemcpyDeviceToDevice, st));
    dst->n += src->n;
    return BDM_OK;
}

bdm_status bdm_sync(bdm_handle h, void *stream) {
    DeviceScope ds__(h);
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    Ctx *c = (Ctx *)h;
    BDM_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    BDM_CUDA_TRY(cudaGetLastError());
    return read_latches(c, true);
}

bdm_status bdm_reserve(bdm_handle h, int64_t max_agents, int64_t nslots) {
    DeviceScope ds__(h);
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    Ctx *c = (Ctx *)h;
    bdm_status s = grow_agents(c, max_agents);
    if (s != BDM_OK) return s;
    return grow_slots(c, nslots);
}

bdm_status bdm_get_stats(bdm_handle h, bdm_stats *out) {
    DeviceScope ds__(h);
    if (!h || !out) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    BDM_CUDA_TRY(cudaMemcpy(c->sc_host, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost));
    out->cand = (int64_t)c->sc_host->stats[0];
    out->nbr = (int64_t)c->sc_host->stats[1];
    out->cont = (int64_t)c->sc_host->stats[2];
    out->n_static = (int64_t)c->sc_host->stats[3];
    out->n_moved = (int64_t)c->sc_host->stats[4];
    out->launches = c->launches;
    return BDM_OK;
}

bdm_status bdm_get_grid_info(bdm_handle h, bdm_grid_info *out) {
    DeviceScope ds__(h);
    if (!h || !out) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    BDM_CUDA_TRY(cudaMemcpy(c->sc_host, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost));
    const DevScalars &s = *c->sc_host;
    out->R = s.R;
    out->L = s.L;
    for (int a = 0; a < 3; ++a) {
        out->origin[a] = s.o[a];
        out->upper[a] = s.hi[a];
        out->dims[a] = s.dims[a];
    }
    out->nslots = s.nslots;
    out->slot_capacity = c->slot_cap;
    return BDM_OK;
}

bdm_status bdm_neighbor_pairs(bdm_handle h, const bdm_agents *a, double radius, uint64_t *pairs,
                              int64_t cap, int64_t *count_host, void *stream) {
    DeviceScope ds__(h);
    if (!h || !count_host) return fail(BDM_EINVAL, "NULL argument");
    if (cap > 0 && !pairs) return fail(BDM_EINVAL, "pairs is NULL");
    Ctx *c = (Ctx *)h;
    bdm_status s = bdm_grid_build(h, a, nullptr, radius, stream);
    if (s != BDM_OK) return s;
    c->grid_valid = false;  // the hook consumes the grid
    *count_host = 0;
    if (a->n == 0) return BDM_OK;
    if ((s = launch_pairs(c, a->n, pairs, cap, (cudaStream_t)stream)) != BDM_OK) return s;
    if ((s = bdm_sync(h, stream)) != BDM_OK) return s;
    unsigned long long cnt = 0;
    BDM_CUDA_TRY(cudaMemcpy(&cnt, c->pair_count, sizeof(cnt), cudaMemcpyDeviceToHost));
    *count_host = (int64_t)cnt;
    if ((int64_t)cnt > cap) return fail(BDM_ECAPACITY, "more pairs than cap");
    return BDM_OK;
}

bdm_status bdm_set_option(bdm_handle h, const char *name, int64_t value) {
    DeviceScope ds__(h);
    if (!h || !name) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    if (strcmp(name, "mech_kernel") == 0) {
        if (value < 0 || value > 5) return fail(BDM_EINVAL, "mech_kernel must be 0..5");
        c->mech_kernel = (int)value;
        return BDM_OK;
    }
    if (strcmp(name, "sir_index_capacity") == 0) {
        if (value < 0) return fail(BDM_EINVAL, "sir_index_capacity must be >= 0");
        c->sir.icap_override = value;
        return BDM_OK;
    }
    if (strcmp(name, "fuse_reduce") == 0) {
        if (value < 0 || value > 1) return fail(BDM_EINVAL, "fuse_reduce must be 0 or 1");
        c->fuse_reduce = (int)value;
        c->fused_valid = false;
        return BDM_OK;
    }
    if (strcmp(name, "diffuse_tma") == 0) {
        if (value < 0 || value > 1) return fail(BDM_EINVAL, "diffuse_tma must be 0 or 1");
        c->diffuse_tma = (int)value;
        return BDM_OK;
    }
    if (strcmp(name, "dense") == 0) {
        if (value < 0 || value > 1) return fail(BDM_EINVAL, "dense must be 0 or 1");
        c->dense = (int)value;
        return BDM_OK;
    }
    if (strcmp(name, "tile_order") == 0) {
        if (value < 0 || value > 1) return fail(BDM_EINVAL, "tile_order must be 0 or 1");
        if (value == c->tile_order) return BDM_OK;
        BDM_CUDA_TRY(cudaDeviceSynchronize());
        uint16_t tab[1024];
        tile_curve((int)value, tab, tab + 512);
        const int32_t v = (int32_t)value;
        BDM_CUDA_TRY(cudaMemcpy(c->sc->hilb, tab, sizeof(tab), cudaMemcpyHostToDevice));
        BDM_CUDA_TRY(cudaMemcpy(&c->sc->tile_order, &v, sizeof(v), cudaMemcpyHostToDevice));
        c->tile_order = (int)value;
        // the slot layout changes: the next build re-sizes the slot array from its geometry
        ctx_free(c, c->box_start);
        ctx_free(c, c->dense_list);
        c->box_start = nullptr;
        c->dense_list = nullptr;
        c->slot_cap = 0;
        c->grid_valid = false;
        return BDM_OK;
    }
    if (strcmp(name, "tile_depth") == 0) {
        if (value < 0 || value > 3) return fail(BDM_EINVAL, "tile_depth must be 0, 1, 2 or 3");
        c->tile_depth = (int)value;
        return BDM_OK;
    }
    if (strcmp(name, "sort_every") == 0) {
        if (value < 0) return fail(BDM_EINVAL, "sort_every must be >= 0");
        c->sort_every = value;
        c->grid_builds = 0;
        return BDM_OK;
    }
    if (strcmp(name, "prefilter") == 0) {
        if (value < 0 || value > 15) return fail(BDM_EINVAL, "prefilter must be 0..15 (bit 0: on; bits 1-2: row-kernel debug paths)");
        c->prefilter = (int)value;
        return BDM_OK;
    }
    return fail(BDM_EINVAL, std::string("unknown option ") + name);
}

int64_t bdm_aura_max_size(int64_t nref, int64_t n) {
    if (nref < 0 || n < 0) return -1;
    return aura_max_size(nref, n);
}

static bdm_status check_aura_agents(const bdm_agents *a, const char *what) {
    if (!a) return fail(BDM_EINVAL, std::string(what) + " is NULL");
    if (a->n < 0 || a->n > a->capacity) return fail(BDM_EINVAL, std::string(what) + ": bad n");
    if (a->n > 0 && (!a->x || !a->y || !a->z || !a->diameter || !a->id || !a->flags))
        return fail(BDM_EINVAL, std::string(what) + ": an array is NULL");
    if (a->n > 0x7FFFFFFFll) return fail(BDM_EINVAL, std::string(what) + ": more than 2^31 - 1 agents");
    return BDM_OK;
}

bdm_status bdm_aura_reference(bdm_handle h, const bdm_agents *msg, bdm_agents *ref, void *stream) {
    DeviceScope ds__(h);
    if (!h) return fail(BDM_EINVAL, "handle is NULL");
    bdm_status s;
    if ((s = check_aura_agents(msg, "msg")) != BDM_OK) return s;
    if (!ref || (msg->n > 0 && (!ref->x || !ref->y || !ref->z || !ref->diameter || !ref->id ||
                                !ref->flags)))
        return fail(BDM_EINVAL, "ref is NULL or an array is NULL");
    if (ref->capacity < msg->n) return fail(BDM_ECAPACITY, "ref capacity < msg->n");
    return launch_aura_reference((Ctx *)h, msg, ref, (cudaStream_t)stream);
}

bdm_status bdm_aura_encode(bdm_handle h, const bdm_agents *msg, const bdm_agents *ref,
                           uint8_t *out, int64_t out_cap, int64_t *out_size_host, void *stream) {
    DeviceScope ds__(h);
    if (!h || !out_size_host) return fail(BDM_EINVAL, "handle or out_size_host is NULL");
    bdm_status s;
    if ((s = check_aura_agents(msg, "msg")) != BDM_OK) return s;
    if ((s = check_aura_agents(ref, "ref")) != BDM_OK) return s;
    if (!out && out_cap > 0) return fail(BDM_EINVAL, "out is NULL");
    return launch_aura_encode((Ctx *)h, msg, ref, out, out_cap, out_size_host, (cudaStream_t)stream);
}

bdm_status bdm_aura_decode(bdm_handle h, const uint8_t *in, int64_t in_size, const bdm_agents *ref,
                           bdm_agents *msg, void *stream) {
    DeviceScope ds__(h);
    if (!h || !in) return fail(BDM_EINVAL, "handle or in is NULL");
    bdm_status s;
    if ((s = check_aura_agents(ref, "ref")) != BDM_OK) return s;
    if (!msg || (msg->capacity > 0 && (!msg->x || !msg->y || !msg->z || !msg->diameter ||
                                       !msg->id || !msg->flags)))
        return fail(BDM_EINVAL, "msg is NULL or an array is NULL");
    return launch_aura_decode((Ctx *)h, in, in_size, ref, msg, (cudaStream_t)stream);
}

bdm_status bdm_tile_curve(int32_t order, uint16_t *rank_out) {
    if (!rank_out) return fail(BDM_EINVAL, "rank_out is NULL");
    if (order < 0 || order > 1) return fail(BDM_EINVAL, "order must be 0 or 1");
    tile_curve((int)order, rank_out, nullptr);
    return BDM_OK;
}

bdm_status bdm_peak_dfma(bdm_handle h, double *dfma_per_s, int32_t *sm_count) {
    DeviceScope ds__(h);
    if (!h || !dfma_per_s || !sm_count) return fail(BDM_EINVAL, "NULL argument");
    Ctx *c = (Ctx *)h;
    *sm_count = c->sm_count;
    return launch_peak_dfma(c->sm_count, dfma_per_s);
}

bdm_status bdm_selftest_recip_div(bdm_handle h, int64_t n, uint64_t seed,
                                  unsigned long long *mismatches) {
    DeviceScope ds__(h);
    if (!h || !mismatches || n <= 0) return fail(BDM_EINVAL, "NULL argument or n <= 0");
    return launch_selftest_recip_div((Ctx *)h, n, seed, mismatches);
}

}  // extern "C"
