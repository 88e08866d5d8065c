// kernels_diffusion.cu -- extracellular diffusion, secretion and chemotaxis (SURVEY 8(f)
// row f4; the paper names diffusion as the next GPU target).
//
//   k_diffuse     Eq. 4.3 (eq:centraldiff), one explicit step, 7-point
//                 stencil with decay; values outside the grid are 0 ("substances
//                 diffuse out of the simulation space"; reading R34);
//                 operation order R35 (no fused multiply-add: -fmad=false)
//   k_secrete     Alg. secretion_module: q into the cell of the agent (R36)
//   k_chemotaxis  Alg. chemotaxis_module: move by weight x the normalized
//                 central-difference gradient at the agent's cell (R37, R38)
//
// The stencil is HBM-bound (8 B read + 8 B written per point and step; ~12 fp64
// operations).  A CTA owns a 32 x 16 column tile and marches a chunk of z planes.
//   k_diffuse_tma  (default; needs nx even for the TMA strides) one thread issues a TMA
//                  3D box load (cp.async.bulk.tensor) of the tile plane with its one-point
//                  halo, 34 x 18 x 1, per z plane into a 4-stage shared-memory ring
//                  signalled by mbarriers; the TMA unit zero-fills the part of the box past
//                  the grid's upper edges (reading R34).  Measured on this B200 + driver
//                  (tools/tma_probe*.cu): a box must start inside the grid and its x start
//                  must be 16-byte aligned (an odd fp64 start or a negative one raises an
//                  illegal instruction).  So the box is 36 x 18 x 1 starting at x = i0 - 2
//                  (0 for the first tile column), y = j0 - 1 (0 for the first tile row), the
//                  plane is indexed relative to that start (the missing low halo is the zero
//                  outside the grid), and planes z = -1, z = nz are not loaded but read as 0
//   k_diffuse      (fallback) the own column's z-1, z, z+1 values in registers, the
//                  current plane in a double-buffered shared tile, the next plane's
//                  values loaded one iteration ahead
// Either way every point is read from HBM once (the x/y halos come from L2).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

constexpr int kFx = 32, kFy = 16;          // tile (points) in x and y
constexpr int kFty = 8;                    // thread rows: each thread owns rows ty, ty + 8
constexpr int kFThreads = kFx * kFty;
constexpr int kFzChunk = 128;              // z planes per work item

struct DiffArgs {
    const double *__restrict__ u;
    double *__restrict__ out;
    int nx, ny, nz;
    int tiles_x, tiles_y, zchunks;
    double decay, cx, cy, cz;
};

__device__ __forceinline__ double ld_or0(const double *__restrict__ u, int nx, int ny, int nz, int i,
                                         int j, int k) {
    return (i >= 0 && j >= 0 && k >= 0 && i < nx && j < ny && k < nz)
               ? u[(size_t)i + (size_t)nx * ((size_t)j + (size_t)ny * (size_t)k)]
               : 0.0;
}

// A column (fixed i, j) read plane by plane: base pointer at plane 0, or null when the
// column lies outside the grid (then every value is 0).
__device__ __forceinline__ double col_at(const double *__restrict__ p, size_t plane, int k, int nz) {
    return (p != nullptr && k >= 0 && k < nz) ? __ldg(p + plane * (size_t)k) : 0.0;
}

__global__ void __launch_bounds__(kFThreads, 4) k_diffuse(DiffArgs A) {
    __shared__ double sp[2][kFy + 2][kFx + 2];   // double-buffered plane with halo
    const int tx = threadIdx.x % kFx, ty = threadIdx.x / kFx;
    const int items = A.tiles_x * A.tiles_y * A.zchunks;
    const size_t plane = (size_t)A.nx * (size_t)A.ny;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int zc = it / (A.tiles_x * A.tiles_y);
        const int t2 = it - zc * A.tiles_x * A.tiles_y;
        const int bj = t2 / A.tiles_x, bi = t2 - bj * A.tiles_x;
        const int i = bi * kFx + tx, j0 = bj * kFy + ty, j1 = j0 + kFty;
        const int z0 = zc * kFzChunk, z1 = min(A.nz, z0 + kFzChunk);
        auto colp = [&](int ci, int cj) -> const double * {
            return (ci >= 0 && cj >= 0 && ci < A.nx && cj < A.ny)
                       ? A.u + (size_t)ci + (size_t)A.nx * (size_t)cj
                       : nullptr;
        };
        const double *p0 = colp(i, j0), *p1 = colp(i, j1);
        // halo columns: x halo for the tile's first / last thread column (both rows),
        // y halo below the tile (thread row 0) and above it (thread row kFty-1)
        const int hxi = tx == 0 ? i - 1 : (tx == kFx - 1 ? i + 1 : -2);
        const double *hx0 = hxi >= -1 ? colp(hxi, j0) : nullptr;
        const double *hx1 = hxi >= -1 ? colp(hxi, j1) : nullptr;
        const bool hxon = (tx == 0 || tx == kFx - 1);
        const int hyj = ty == 0 ? bj * kFy - 1 : (ty == kFty - 1 ? bj * kFy + kFy : -2);
        const bool hyon = (ty == 0 || ty == kFty - 1);
        const double *hy = hyon ? colp(i, hyj) : nullptr;
        const int hcol = tx == 0 ? 0 : kFx + 1;        // x-halo column in the plane
        const int hrow = ty == 0 ? 0 : kFy + 1;         // y-halo row in the plane
        double zm0 = col_at(p0, plane, z0 - 1, A.nz), zm1 = col_at(p1, plane, z0 - 1, A.nz);
        double c0 = col_at(p0, plane, z0, A.nz), c1 = col_at(p1, plane, z0, A.nz);
        double hx0v = col_at(hx0, plane, z0, A.nz), hx1v = col_at(hx1, plane, z0, A.nz);
        double hyv = col_at(hy, plane, z0, A.nz);
        double *const o0 = (p0 != nullptr) ? A.out + (size_t)i + (size_t)A.nx * (size_t)j0 : nullptr;
        double *const o1 = (p1 != nullptr) ? A.out + (size_t)i + (size_t)A.nx * (size_t)j1 : nullptr;
        int b = 0;
        for (int z = z0; z < z1; ++z, b ^= 1) {
            // next plane, one iteration ahead
            const double zp0 = col_at(p0, plane, z + 1, A.nz), zp1 = col_at(p1, plane, z + 1, A.nz);
            const double hx0n = col_at(hx0, plane, z + 1, A.nz), hx1n = col_at(hx1, plane, z + 1, A.nz);
            const double hyn = col_at(hy, plane, z + 1, A.nz);
            sp[b][ty + 1][tx + 1] = c0;
            sp[b][ty + 1 + kFty][tx + 1] = c1;
            if (hxon) {
                sp[b][ty + 1][hcol] = hx0v;
                sp[b][ty + 1 + kFty][hcol] = hx1v;
            }
            if (hyon) sp[b][hrow][tx + 1] = hyv;
            __syncthreads();  // one barrier per plane: the next plane goes to the other buffer
            // Eq. 4.3 in the order of reading R35
            if (o0 != nullptr) {
                double v = c0 * A.decay;
                v = v + A.cx * ((sp[b][ty + 1][tx + 2] - 2.0 * c0) + sp[b][ty + 1][tx]);
                v = v + A.cy * ((sp[b][ty + 2][tx + 1] - 2.0 * c0) + sp[b][ty][tx + 1]);
                v = v + A.cz * ((zp0 - 2.0 * c0) + zm0);
                o0[plane * (size_t)z] = v;
            }
            if (o1 != nullptr) {
                const int r = ty + 1 + kFty;
                double v = c1 * A.decay;
                v = v + A.cx * ((sp[b][r][tx + 2] - 2.0 * c1) + sp[b][r][tx]);
                v = v + A.cy * ((sp[b][r + 1][tx + 1] - 2.0 * c1) + sp[b][r - 1][tx + 1]);
                v = v + A.cz * ((zp1 - 2.0 * c1) + zm1);
                o1[plane * (size_t)z] = v;
            }
            zm0 = c0;
            zm1 = c1;
            c0 = zp0;
            c1 = zp1;
            hx0v = hx0n;
            hx1v = hx1n;
            hyv = hyn;
        }
        __syncthreads();  // the next work item reuses both buffers
    }
}

// ------------------------------------------------------------------ TMA version
constexpr int kTS = 4;                                   // plane stages
constexpr int kTBx = kFx + 4, kTBy = kFy + 2;            // TMA box (x start even, see above)
constexpr int kTPlane = kTBy * kTBx;                     // doubles per staged plane
constexpr int kTStride = ((kTPlane * 8 + 127) / 128) * 128;  // bytes per stage (128-aligned)
constexpr int kTSmem = kTS * kTStride + kTS * 8;

__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "DWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra DWAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(kFThreads) k_diffuse_tma(const __grid_constant__ CUtensorMap tm,
                                                          DiffArgs A) {
    extern __shared__ __align__(128) unsigned char dsm[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t bars = sbase + kTS * kTStride;
    const int tid = threadIdx.x, tx = tid % kFx, ty = tid / kFx;
    if (tid == 0) {
        for (int s = 0; s < kTS; ++s) mbar_init1(bars + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int items = A.tiles_x * A.tiles_y * A.zchunks;
    const size_t plane = (size_t)A.nx * (size_t)A.ny;
    uint32_t pcount = 0;  // planes issued by this CTA so far (stage / parity bookkeeping)
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int zc = it / (A.tiles_x * A.tiles_y);
        const int t2 = it - zc * A.tiles_x * A.tiles_y;
        const int bj = t2 / A.tiles_x, bi = t2 - bj * A.tiles_x;
        const int i0 = bi * kFx, jt = bj * kFy;
        const int z0 = zc * kFzChunk, z1 = min(A.nz, z0 + kFzChunk);
        const int nplanes = (z1 - z0) + 2;  // planes z0-1 .. z1 (q = 0 .. nplanes-1)
        // box start (x even and >= 0, y >= 0); the plane is indexed relative to it
        const int sx = i0 >= 2 ? i0 - 2 : 0, sy = jt >= 1 ? jt - 1 : 0;
        // issue plane q (z = z0 - 1 + q) into its stage; the part past the upper grid
        // edges is zero-filled by the TMA unit; planes outside [0, nz) are not loaded (a
        // plain arrival completes the stage's phase) and read as zero
        auto issue = [&](int q) {
            const uint32_t G = pcount + (uint32_t)q, s = G % kTS;
            const uint32_t bar = bars + 8 * s, dst = sbase + s * kTStride;
            const int z = z0 - 1 + q;
            if (z < 0 || z >= A.nz) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
                return;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"(kTPlane * 8)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(sx), "r"(sy), "r"(z), "r"(bar)
                : "memory");
        };
        auto wait = [&](int q) {
            const uint32_t G = pcount + (uint32_t)q;
            mbar_wait_parity(bars + 8 * (G % kTS), (G / kTS) & 1u);
        };
        auto at = [&](int q, int y, int x) -> double {  // staged plane q, grid point (x, y)
            const uint32_t G = pcount + (uint32_t)q;
            const double *p = reinterpret_cast<const double *>(dsm + (G % kTS) * kTStride);
            return p[(y - sy) * kTBx + (x - sx)];
        };
        if (tid == 0)
            for (int q = 0; q < 3 && q < nplanes; ++q) issue(q);
        wait(0);
        wait(1);
        const int i = i0 + tx, j0 = jt + ty, j1 = j0 + kFty;
        const bool own0 = i < A.nx && j0 < A.ny, own1 = i < A.nx && j1 < A.ny;
        double *const o0 = A.out + (size_t)i + (size_t)A.nx * (size_t)j0;
        double *const o1 = A.out + (size_t)i + (size_t)A.nx * (size_t)j1;
        for (int z = z0; z < z1; ++z) {
            const int qc = z - z0 + 1;  // centre plane
            if (tid == 0 && qc + 2 < nplanes) issue(qc + 2);
            wait(qc + 1);
            const bool hzb = z > 0, hza = z + 1 < A.nz;
            // Eq. 4.3 in the order of reading R35; neighbours left of / below the grid are 0
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = h ? j1 : j0;
                if (!(h ? own1 : own0)) continue;
                const double c = at(qc, j, i);
                const double xl = i > 0 ? at(qc, j, i - 1) : 0.0, xr = at(qc, j, i + 1);
                const double yl = j > 0 ? at(qc, j - 1, i) : 0.0, yr = at(qc, j + 1, i);
                const double zl = hzb ? at(qc - 1, j, i) : 0.0;
                const double zr = hza ? at(qc + 1, j, i) : 0.0;
                double v = c * A.decay;
                v = v + A.cx * ((xr - 2.0 * c) + xl);
                v = v + A.cy * ((yr - 2.0 * c) + yl);
                v = v + A.cz * ((zr - 2.0 * c) + zl);
                (h ? o1 : o0)[plane * (size_t)z] = v;
            }
            __syncthreads();  // everyone is done with plane qc - 1 before its stage refills
        }
        pcount += (uint32_t)nplanes;
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

bdm_status launch_diffuse(Ctx *c, const double *u_in, double *u_out, const bdm_grid3 *g,
                          double nu, double mu, double dt, cudaStream_t st) {
    if (g->nx <= 0 || g->ny <= 0 || g->nz <= 0) return BDM_OK;
    static int per_sm_dev[kMaxDevices] = {};
    int &per_sm = per_sm_dev[c->device];
    if (!per_sm) {
        int v = 0;
        BDM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_diffuse, kFThreads, 0));
        per_sm = v < 1 ? 1 : v;
    }
    DiffArgs A;
    A.u = u_in;
    A.out = u_out;
    A.nx = (int)g->nx;
    A.ny = (int)g->ny;
    A.nz = (int)g->nz;
    A.tiles_x = (A.nx + kFx - 1) / kFx;
    A.tiles_y = (A.ny + kFy - 1) / kFy;
    A.zchunks = (A.nz + kFzChunk - 1) / kFzChunk;
    A.decay = 1.0 - mu * dt;
    A.cx = (nu * dt) / (g->dx * g->dx);
    A.cy = (nu * dt) / (g->dy * g->dy);
    A.cz = (nu * dt) / (g->dz * g->dz);
    const long long items = (long long)A.tiles_x * A.tiles_y * A.zchunks;
    // TMA path: global strides must be multiples of 16 B (nx even), coordinates < 2^31;
    // grids narrower than one box take the other kernel
    PFN_cuTensorMapEncodeTiled_v12000 enc = c->diffuse_tma ? tensor_map_encoder() : nullptr;
    if (enc && (A.nx % 2) == 0 && A.nx >= kTBx && A.ny >= kTBy) {
        static int per_sm_t_dev[kMaxDevices] = {};
        int &per_sm_t = per_sm_t_dev[c->device];
        if (!per_sm_t) {
            BDM_CUDA_TRY(cudaFuncSetAttribute(k_diffuse_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kTSmem));
            int v = 0;
            BDM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_diffuse_tma,
                                                                       kFThreads, kTSmem));
            per_sm_t = v < 1 ? 1 : v;
        }
        CUtensorMap tm;
        const cuuint64_t gdim[3] = {(cuuint64_t)A.nx, (cuuint64_t)A.ny, (cuuint64_t)A.nz};
        const cuuint64_t gstr[2] = {(cuuint64_t)A.nx * 8, (cuuint64_t)A.nx * (cuuint64_t)A.ny * 8};
        const cuuint32_t box[3] = {kTBx, kTBy, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(u_in),
                               gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r == CUDA_SUCCESS) {
            const long long slots = (long long)c->sm_count * per_sm_t;
            k_diffuse_tma<<<(unsigned)(items < slots ? items : slots), kFThreads, kTSmem, st>>>(tm, A);
            c->launches += 1;
            BDM_LAUNCH_CHECK("k_diffuse_tma");
            return BDM_OK;
        }
    }
    const long long slots = (long long)c->sm_count * per_sm;
    k_diffuse<<<(unsigned)(items < slots ? items : slots), kFThreads, 0, st>>>(A);
    c->launches += 1;
    BDM_LAUNCH_CHECK("k_diffuse");
    return BDM_OK;
}

// ------------------------------------------------------------------ agents <-> grid
struct GridView3 {
    int nx, ny, nz;
    double lo0, lo1, lo2, dx, dy, dz;
};

__device__ __forceinline__ int cell_of(double p, double lo, double d, int n) {
    double b = floor((p - lo) / d);
    b = b < 0.0 ? 0.0 : b;
    b = b > (double)(n - 1) ? (double)(n - 1) : b;
    return (int)b;
}

__global__ void k_secrete(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                          const double *__restrict__ z, const uint8_t *__restrict__ type,
                          int type_sel, double q, double *__restrict__ u, GridView3 g) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n || (int)type[a] != type_sel) return;
    const int i = cell_of(x[a], g.lo0, g.dx, g.nx), j = cell_of(y[a], g.lo1, g.dy, g.ny),
              k = cell_of(z[a], g.lo2, g.dz, g.nz);
    // every agent adds the same q, so the sequence of partial sums (and the result) does
    // not depend on the order of the atomic additions
    atomicAdd(&u[(size_t)i + (size_t)g.nx * ((size_t)j + (size_t)g.ny * (size_t)k)], q);
}

__global__ void k_chemotaxis(int64_t n, double *__restrict__ x, double *__restrict__ y,
                             double *__restrict__ z, const uint8_t *__restrict__ type, int type_sel,
                             double weight, const double *__restrict__ u, GridView3 g) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n || (int)type[a] != type_sel) return;
    const double px = x[a], py = y[a], pz = z[a];
    const int i = cell_of(px, g.lo0, g.dx, g.nx), j = cell_of(py, g.lo1, g.dy, g.ny),
              k = cell_of(pz, g.lo2, g.dz, g.nz);
    const double gx = (ld_or0(u, g.nx, g.ny, g.nz, i + 1, j, k) - ld_or0(u, g.nx, g.ny, g.nz, i - 1, j, k)) /
                      (2.0 * g.dx);
    const double gy = (ld_or0(u, g.nx, g.ny, g.nz, i, j + 1, k) - ld_or0(u, g.nx, g.ny, g.nz, i, j - 1, k)) /
                      (2.0 * g.dy);
    const double gz = (ld_or0(u, g.nx, g.ny, g.nz, i, j, k + 1) - ld_or0(u, g.nx, g.ny, g.nz, i, j, k - 1)) /
                      (2.0 * g.dz);
    const double n2 = gx * gx + gy * gy + gz * gz;
    if (!(n2 > 0.0)) return;
    const double nrm = sqrt(n2);
    x[a] = px + weight * (gx / nrm);
    y[a] = py + weight * (gy / nrm);
    z[a] = pz + weight * (gz / nrm);
}

static GridView3 view_of(const bdm_grid3 *g) {
    GridView3 v;
    v.nx = (int)g->nx;
    v.ny = (int)g->ny;
    v.nz = (int)g->nz;
    v.lo0 = g->lo[0];
    v.lo1 = g->lo[1];
    v.lo2 = g->lo[2];
    v.dx = g->dx;
    v.dy = g->dy;
    v.dz = g->dz;
    return v;
}

bdm_status launch_secrete(Ctx *c, const bdm_agents *a, const uint8_t *type, int type_sel, double q,
                          double *u, const bdm_grid3 *g, cudaStream_t st) {
    if (a->n == 0) return BDM_OK;
    k_secrete<<<(unsigned)((a->n + 255) / 256), 256, 0, st>>>(a->n, a->x, a->y, a->z, type,
                                                              type_sel, q, u, view_of(g));
    c->launches += 1;
    BDM_LAUNCH_CHECK("k_secrete");
    return BDM_OK;
}

bdm_status launch_chemotaxis(Ctx *c, bdm_agents *a, const uint8_t *type, int type_sel,
                             double weight, const double *u, const bdm_grid3 *g, cudaStream_t st) {
    if (a->n == 0) return BDM_OK;
    k_chemotaxis<<<(unsigned)((a->n + 255) / 256), 256, 0, st>>>(a->n, a->x, a->y, a->z, type,
                                                                 type_sel, weight, u, view_of(g));
    c->launches += 1;
    BDM_LAUNCH_CHECK("k_chemotaxis");
    return BDM_OK;
}

}  // namespace bdm
