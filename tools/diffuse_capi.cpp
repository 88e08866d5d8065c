// Calls bdm_diffuse through the C ABI only (no PyTorch in the process).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "bdm.h"

int main(int argc, char **argv) {
    const int64_t nx = 64, ny = 48, nz = 4;
    bdm_handle h;
    if (bdm_create(&h, 0, 16) != BDM_OK) { printf("create: %s\n", bdm_last_error()); return 1; }
    if (argc > 1) bdm_set_option(h, "diffuse_tma", atoi(argv[1]));
    double *u, *v;
    cudaMalloc(&u, nx * ny * nz * 8);
    cudaMalloc(&v, nx * ny * nz * 8);
    std::vector<double> hu(nx * ny * nz, 1.0);
    cudaMemcpy(u, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice);
    bdm_grid3 g = {nx, ny, nz, {0, 0, 0}, 1.0, 1.0, 1.0};
    bdm_status s = bdm_diffuse(h, u, v, &g, 0.1, 0.0, 0.5, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %d sync %s\n", (int)s, cudaGetErrorString(e));
    std::vector<double> hv(hu.size());
    cudaMemcpy(hv.data(), v, hv.size() * 8, cudaMemcpyDeviceToHost);
    printf("v[0]=%g v[mid]=%g\n", hv[0], hv[nx + nx * ny]);
    return e == cudaSuccess ? 0 : 1;
}
