// Probe 2: the k_diffuse_tma instruction mix in isolation.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void wait_par(uint32_t bar, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(par) : "memory");
}

// mode 0: plain arrive with sink, then wait.  mode 1: plain arrive with a state register.
// mode 2: TMA (valid coords) through a lambda, 4-stage ring, 8 planes.
__global__ void probe2(const __grid_constant__ CUtensorMap tm, int mode, double *out) {
    extern __shared__ __align__(128) unsigned char dsm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t bars = sb + 4 * 4992;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (mode == 0) {
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bars) : "memory");
        wait_par(bars, 0);
    } else if (mode == 1) {
        if (threadIdx.x == 0) {
            uint64_t st;
            asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(bars) : "memory");
        }
        wait_par(bars, 0);
    } else {
        auto issue = [&](int q) {
            const uint32_t s = q % 4, bar = bars + 8 * s, dst = sb + s * 4992;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4896) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(q), "r"(bar) : "memory");
        };
        if (threadIdx.x == 0) for (int q = 0; q < 3; ++q) issue(q);
        double acc = 0.0;
        for (int q = 0; q < 8; ++q) {
            if (threadIdx.x == 0 && q + 3 < 8) issue(q + 3);
            wait_par(bars + 8 * (q % 4), (q / 4) & 1);
            acc += reinterpret_cast<const double *>(dsm + (q % 4) * 4992)[threadIdx.x];
            __syncthreads();
        }
        out[threadIdx.x] = acc;
    }
}

int main() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    const int nx = 64, ny = 48, nz = 16;
    double *d, *o;
    cudaMalloc(&d, (size_t)nx * ny * nz * 8);
    cudaMemset(d, 0, (size_t)nx * ny * nz * 8);
    cudaMalloc(&o, 4096 * 8);
    CUtensorMap tm;
    cuuint64_t gdim[3] = {nx, ny, nz};
    cuuint64_t gstr[2] = {nx * 8, (cuuint64_t)nx * ny * 8};
    cuuint32_t box[3] = {34, 18, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    for (int mode = 2; mode >= 0; --mode) {
        probe2<<<1, 256, 20000>>>(tm, mode, o);
        cudaError_t k = cudaDeviceSynchronize();
        printf("mode %d encode %d: %s\n", mode, (int)r, cudaGetErrorString(k));
        if (k != cudaSuccess) return 1;
    }
    return 0;
}
