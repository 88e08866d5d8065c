// Standalone TMA probe: 3D box loads (fp64) with positive / negative start coordinates.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tm, double *out, int x0, int y0, int z0,
                      int nbytes) {
    __shared__ __align__(128) double buf[2048];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(buf);
    const unsigned bb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(nbytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(sb), "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(x0), "r"(y0), "r"(z0), "r"(bb) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(bb) : "memory");
    for (int k = threadIdx.x; k < nbytes / 8; k += blockDim.x) out[k] = buf[k];
}

int main() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    printf("entry point: %d %d %p\n", (int)e, (int)q, p);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    const int nx = 64, ny = 48, nz = 8;
    std::vector<double> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 2048 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    struct Case { int bx, by, x0, y0, z0; } cases[] = {
        {32, 16, 0, 0, 0}, {34, 18, 0, 0, 1}, {34, 18, 40, 40, 7}, {34, 18, 31, 31, 8}, {34, 18, 63, 47, 3}, {34, 18, 64, 0, 2}};
    for (auto c : cases) {
        CUtensorMap tm;
        cuuint64_t gdim[3] = {nx, ny, nz};
        cuuint64_t gstr[2] = {nx * 8, (cuuint64_t)nx * ny * 8};
        cuuint32_t box[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, gdim, gstr, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaMemset(o, 0xff, 2048 * 8);
        probe<<<1, 128>>>(tm, o, c.x0, c.y0, c.z0, c.bx * c.by * 8);
        cudaError_t k = cudaDeviceSynchronize();
        std::vector<double> r2(c.bx * c.by);
        cudaMemcpy(r2.data(), o, r2.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < c.by; ++yy)
            for (int xx = 0; xx < c.bx; ++xx) {
                int gx = c.x0 + xx, gy = c.y0 + yy, gz = c.z0;
                double want = (gx >= 0 && gy >= 0 && gz >= 0 && gx < nx && gy < ny && gz < nz) ? h[gx + nx * (gy + ny * gz)] : 0.0;
                if (r2[xx + c.bx * yy] != want) ++bad;
            }
        printf("box %dx%d at (%d,%d,%d): encode %d kernel %s mismatches %d\n", c.bx, c.by, c.x0, c.y0, c.z0, (int)r, cudaGetErrorString(k), bad);
        if (k != cudaSuccess) return 1;
    }
    return 0;
}
