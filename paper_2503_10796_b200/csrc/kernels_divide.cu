// kernels_divide.cu -- growth + division with add-compaction.
//
// Alg. 4's control flow "grow while the diameter is below the maximum, else divide"
// (algo:tumor_growth_module) with division probability 1; Cell::Divide
// (P:7823-7831): volume ratio 0.5, daughter placed along the division axis; agent
// additions are committed in parallel at the end of the iteration and
// become visible at the next one.  Readings R13-R15, R28.
//
//   k_div_mark   flag[id] = (V >= v_max), one per agent, indexed by the dense id
//   scan         exclusive scan over n + 1 flags -> rank of each divider in id order
//                and the total (the paper's "total number of additions")
//   k_div_apply  growth, or division: mother keeps its slot, the daughter is appended
//                at n + rank with id n + rank (all-or-nothing on capacity)
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

// cbrt_det (R28) and division_axis (R13) live in bdm_internal.cuh (shared with row f2).

__global__ void __launch_bounds__(256) k_div_mark(int64_t n, const double *__restrict__ vol,
                                                  const uint32_t *__restrict__ id, double v_max,
                                                  uint32_t *__restrict__ flag_by_id,
                                                  DevScalars *__restrict__ sc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const uint32_t me = id[i];
        if ((int64_t)me < n) flag_by_id[me] = (vol[i] < v_max) ? 0u : 1u;
        else sc->overflow = 5;  // ids must be exactly 0..n-1: nothing is modified
    }
    if (i == 0) flag_by_id[n] = 0u;
}

__global__ void __launch_bounds__(256) k_div_apply(
    int64_t n, int64_t capacity, double *__restrict__ x, double *__restrict__ y,
    double *__restrict__ z, double *__restrict__ d, double *__restrict__ vol,
    uint32_t *__restrict__ id, uint32_t *__restrict__ flags,
    const uint32_t *__restrict__ rank_by_id, double growth, double v_max, double vol_to_r3,
    uint32_t k0, uint32_t k1, uint32_t step, DevScalars *__restrict__ sc,
    long long *__restrict__ n_new) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sc->overflow == 5) {  // an id outside 0..n-1 (k_div_mark): no change
        if (i == 0) *n_new = (long long)n;
        return;
    }
    const int64_t total = (int64_t)rank_by_id[n];
    if (n + total > capacity) {  // all-or-nothing: nothing is modified
        if (i == 0) {
            sc->overflow = 2;
            *n_new = -(long long)(n + total);
        }
        return;
    }
    if (i == 0) *n_new = (long long)(n + total);
    if (i >= n) return;
    const double V = vol[i];
    if (V < v_max) {  // grow (Alg. 4 line "IncreaseVolume")
        const double Vn = V + growth;
        const double dn = 2.0 * cbrt_det(Vn * vol_to_r3);
        if (dn > d[i]) flags[i] |= BDM_FLAG_GREW;
        vol[i] = Vn;
        d[i] = dn;
    } else {          // divide (Cell::Divide, volume ratio 0.5)
        const uint32_t me = id[i];
        const int64_t j = n + (int64_t)rank_by_id[me];
        const double Vh = V * 0.5;
        const double r = cbrt_det(Vh * vol_to_r3);
        double ux, uy, uz;
        division_axis(k0, k1, me, step, ux, uy, uz);
        const double px = x[i], py = y[i], pz = z[i];
        x[i] = px - r * ux;
        y[i] = py - r * uy;
        z[i] = pz - r * uz;
        x[j] = px + r * ux;
        y[j] = py + r * uy;
        z[j] = pz + r * uz;
        vol[i] = Vh;
        vol[j] = Vh;
        d[i] = 2.0 * r;
        d[j] = 2.0 * r;
        flags[i] |= BDM_FLAG_MOVED;
        flags[j] = BDM_FLAG_ADDED;
        id[j] = (uint32_t)j;
    }
}

bdm_status launch_grow_divide(Ctx *c, bdm_agents *a, double growth, double v_max, double vol_to_r3,
                              uint64_t seed, uint32_t step, long long *n_new_host,
                              cudaStream_t st) {
    const int64_t n = a->n;
    const unsigned nb = (unsigned)((n + 256) / 256);
    {
        const bdm_status s0 = need_agent_buf(c, &c->div_rank);
        if (s0 != BDM_OK) return s0;
    }
    k_div_mark<<<nb, 256, 0, st>>>(n, a->volume, a->id, v_max, c->div_rank, c->sc);
    BDM_LAUNCH_CHECK("k_div_mark");
    bdm_status s = launch_scan_u32(c, c->div_rank, n + 1, st);
    if (s != BDM_OK) return s;
    k_div_apply<<<nb, 256, 0, st>>>(n, a->capacity, a->x, a->y, a->z, a->diameter, a->volume,
                                    a->id, a->flags, c->div_rank, growth, v_max, vol_to_r3,
                                    (uint32_t)seed, (uint32_t)(seed >> 32), step, c->sc,
                                    c->n_new);
    BDM_LAUNCH_CHECK("k_div_apply");
    BDM_CUDA_TRY(cudaMemcpyAsync(n_new_host, c->n_new, sizeof(long long), cudaMemcpyDeviceToHost, st));
    c->launches += 2;
    return BDM_OK;
}

}  // namespace bdm
