// The library's kernels_diffusion.cu compiled standalone, to bisect compile flags.
#include "../paper_2503_10796_b200/csrc/kernels_diffusion.cu"
#include <cstdio>
#include <vector>
namespace bdm {
void set_error(const std::string &msg) { printf("error: %s\n", msg.c_str()); }
bdm_status cuda_fail(cudaError_t e, const char *what) { printf("cuda: %s %s\n", what, cudaGetErrorString(e)); return BDM_ECUDA; }
}
int main() {
    bdm::Ctx c;
    c.sm_count = 148;
    const int64_t nx = 64, ny = 48, nz = 4;
    double *u, *v;
    cudaMalloc(&u, nx * ny * nz * 8);
    cudaMalloc(&v, nx * ny * nz * 8);
    std::vector<double> hu(nx * ny * nz, 1.0);
    cudaMemcpy(u, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice);
    bdm_grid3 g = {nx, ny, nz, {0, 0, 0}, 1.0, 1.0, 1.0};
    bdm_status s = bdm::launch_diffuse(&c, u, v, &g, 0.1, 0.0, 0.5, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %d sync %s\n", (int)s, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
