// kernels_onco.cu -- oncology behaviour with agent removal.
//
// Alg. 4 (algo:tumor_growth_module) with the Table 4.2 parameters
// on agents carrying their post-mechanics state, and the parallel agent
// removal of sec. "Agent addition and removal".  Readings R41-R45
// (DESIGN.md): unit-vector Brownian step; Philox counters (id, step, 5) for movement and
// death and (id, step, 6) for division; growth as R28, division as R13; removal keeps
// the survivors' order, daughters follow in mother-id order with ids id_next + rank.
//
//   k_onco_decide  per agent: dead (age gate + p_death) -> keep[i] = 0; divider
//                  (d >= d_max, p_div) -> divf[id] = 1 (ids are sparse after removals,
//                  so the flags are indexed by id over [0, id_next))
//   scans          keep -> survivor slot (the paper's compaction of the vector);
//                  divf -> rank of each divider in id order (and the totals)
//   k_onco_apply   survivors: Brownian move, age, growth or division, written to the
//                  workspace at their survivor slot, daughters at nsurv + rank;
//                  all-or-nothing on capacity.  Ages are a property table indexed by
//                  id (the mechanics step reorders the SoA; ids travel with it)
//   k_onco_copy    workspace -> caller arrays
// The paper removes by swapping the last agents into the holes (Fig. 5.1); a
// stable compaction is the GPU-natural equivalent, and memory order never enters a
// result (R32).
#include <cuda_runtime.h>
#include <math.h>

#include "bdm_internal.cuh"

namespace bdm {

struct OncoArgs {
    int64_t n, capacity, id_next;
    double *__restrict__ x;
    double *__restrict__ y;
    double *__restrict__ z;
    double *__restrict__ d;
    double *__restrict__ vol;
    uint32_t *__restrict__ id;
    uint32_t *__restrict__ flags;
    uint32_t *__restrict__ age;    // indexed by id
    int64_t age_cap;
    // workspace
    double *__restrict__ wx;
    double *__restrict__ wy;
    double *__restrict__ wz;
    double *__restrict__ wd;
    double *__restrict__ wvol;
    uint32_t *__restrict__ wid;
    uint32_t *__restrict__ wflags;
    uint32_t *__restrict__ keep;   // n + 1, scanned in place
    uint32_t *__restrict__ divf;   // id_next + 1, scanned in place
    long long *__restrict__ out;   // [new n, new id_next]
    double rate, growth, dmax, p_death, p_div, vol_to_r3;
    uint32_t min_age, k0, k1, step;
};

__global__ void __launch_bounds__(256) k_onco_decide(OncoArgs A) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) A.keep[A.n] = 0u;
    if (i >= A.n) return;
    const uint32_t me = A.id[i];
    const U4 w = philox10(me, 0u, A.step, 5u, A.k0, A.k1);
    const bool dead = A.age[me] >= A.min_age && uniform32(w.d) < A.p_death;
    A.keep[i] = dead ? 0u : 1u;
    if (!dead && !(A.d[i] < A.dmax)) {
        const U4 v = philox10(me, 0u, A.step, 6u, A.k0, A.k1);
        if (uniform32(v.a) < A.p_div) A.divf[me] = 1u;
    }
}

__global__ void __launch_bounds__(256) k_onco_apply(OncoArgs A, DevScalars *__restrict__ sc) {
    const int64_t nsurv = (int64_t)A.keep[A.n], ndiv = (int64_t)A.divf[A.id_next];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nsurv + ndiv > A.capacity || A.id_next + ndiv > A.age_cap) {
        // all-or-nothing: the caller's arrays stay as they are
        if (i == 0) {
            sc->overflow = 2;
            A.out[0] = -(long long)(nsurv + ndiv);
            A.out[1] = (long long)A.id_next;
        }
        return;
    }
    if (i == 0) {
        A.out[0] = (long long)(nsurv + ndiv);
        A.out[1] = (long long)(A.id_next + ndiv);
    }
    if (i >= A.n) return;
    const uint32_t k = A.keep[i];
    if (A.keep[i + 1] == k) return;  // removed (the scan did not advance)
    const uint32_t me = A.id[i];
    const U4 w = philox10(me, 0u, A.step, 5u, A.k0, A.k1);
    double px = A.x[i], py = A.y[i], pz = A.z[i];
    uint32_t fl = A.flags[i];
    // Alg. 4: brownian = v / |v| (R41)
    const double vx = 2.0 * uniform32(w.a) - 1.0;
    const double vy = 2.0 * uniform32(w.b) - 1.0;
    const double vz = 2.0 * uniform32(w.c) - 1.0;
    const double n2 = vx * vx + vy * vy + vz * vz;
    if (n2 > 0.0) {
        const double nv = sqrt(n2);
        px = px + (vx / nv) * A.rate;
        py = py + (vy / nv) * A.rate;
        pz = pz + (vz / nv) * A.rate;
        if (A.rate != 0.0) fl |= BDM_FLAG_MOVED;
    }
    double dd = A.d[i], V = A.vol[i];
    if (dd < A.dmax) {  // grow (R43 = R28)
        const double Vn = V + A.growth;
        const double dn = 2.0 * cbrt_det(Vn * A.vol_to_r3);
        if (dn > dd) fl |= BDM_FLAG_GREW;
        V = Vn;
        dd = dn;
    } else if (A.divf[me + 1] != A.divf[me]) {  // divide (R43 = R13)
        const uint32_t rank = A.divf[me];
        const int64_t j = nsurv + (int64_t)rank;
        const double Vh = V * 0.5;
        const double r = cbrt_det(Vh * A.vol_to_r3);
        double ux, uy, uz;
        division_axis(A.k0, A.k1, me, A.step, ux, uy, uz);
        A.wx[j] = px + r * ux;
        A.wy[j] = py + r * uy;
        A.wz[j] = pz + r * uz;
        A.wd[j] = 2.0 * r;
        A.wvol[j] = Vh;
        A.wid[j] = (uint32_t)(A.id_next + (int64_t)rank);
        A.wflags[j] = BDM_FLAG_ADDED;
        A.age[A.id_next + (int64_t)rank] = 0u;
        px = px - r * ux;
        py = py - r * uy;
        pz = pz - r * uz;
        V = Vh;
        dd = 2.0 * r;
        fl |= BDM_FLAG_MOVED;
    }
    A.wx[k] = px;
    A.wy[k] = py;
    A.wz[k] = pz;
    A.wd[k] = dd;
    A.wvol[k] = V;
    A.wid[k] = me;
    A.wflags[k] = fl;
    A.age[me] = A.age[me] + 1u;
}

__global__ void __launch_bounds__(256) k_onco_copy(OncoArgs A) {
    const long long m = A.out[0];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        A.x[k] = A.wx[k];
        A.y[k] = A.wy[k];
        A.z[k] = A.wz[k];
        A.d[k] = A.wd[k];
        A.vol[k] = A.wvol[k];
        A.id[k] = A.wid[k];
        A.flags[k] = A.wflags[k];
    }
}

bdm_status launch_onco_step(Ctx *c, bdm_agents *a, uint32_t *age, int64_t age_cap,
                            const bdm_onco_params *p, int64_t id_next, long long *out_host,
                            cudaStream_t st) {
    const int64_t n = a->n;
    if ((int64_t)c->onco_id_cap < id_next + 1) {
        BDM_CUDA_TRY(cudaStreamSynchronize(st));
        if (c->onco_id) cudaFree(c->onco_id);
        c->onco_id = nullptr;
        const int64_t cap = id_next + id_next / 4 + 1024;
        BDM_CUDA_TRY(cudaMalloc(&c->onco_id, (size_t)cap * sizeof(uint32_t)));
        c->onco_id_cap = cap;
    }
    {
        bdm_status s0;
        if ((s0 = need_agent_buf(c, &c->svol)) != BDM_OK) return s0;
        if ((s0 = need_agent_buf(c, &c->lrank)) != BDM_OK) return s0;
    }
    if (!c->onco_out) BDM_CUDA_TRY(cudaMalloc(&c->onco_out, 2 * sizeof(long long)));
    OncoArgs A;
    A.n = n;
    A.capacity = a->capacity;
    A.id_next = id_next;
    A.x = a->x; A.y = a->y; A.z = a->z; A.d = a->diameter; A.vol = a->volume;
    A.id = a->id; A.flags = a->flags; A.age = age; A.age_cap = age_cap;
    A.wx = c->sx; A.wy = c->sy; A.wz = c->sz; A.wd = c->sd; A.wvol = c->svol;
    A.wid = c->sidf; A.wflags = c->sflags;
    A.keep = c->lrank;
    A.divf = c->onco_id;
    A.out = c->onco_out;
    A.rate = p->displacement_rate;
    A.growth = p->growth;
    A.dmax = p->max_diameter;
    A.p_death = p->p_death;
    A.p_div = p->p_div;
    A.vol_to_r3 = 0.75 / M_PI;  // r^3 = V * 0.75/pi, computed once (R28)
    A.min_age = p->min_age;
    A.k0 = (uint32_t)p->seed;
    A.k1 = (uint32_t)(p->seed >> 32);
    A.step = p->step;
    BDM_CUDA_TRY(cudaMemsetAsync(c->onco_id, 0, (size_t)(id_next + 1) * sizeof(uint32_t), st));
    const unsigned nb = (unsigned)((n + 256) / 256);
    k_onco_decide<<<nb, 256, 0, st>>>(A);
    BDM_LAUNCH_CHECK("k_onco_decide");
    bdm_status s = launch_scan_u32(c, c->lrank, n + 1, st);
    if (s != BDM_OK) return s;
    if ((s = launch_scan_u32(c, c->onco_id, id_next + 1, st)) != BDM_OK) return s;
    k_onco_apply<<<nb, 256, 0, st>>>(A, c->sc);
    BDM_LAUNCH_CHECK("k_onco_apply");
    k_onco_copy<<<(unsigned)(c->sm_count * 8), 256, 0, st>>>(A);
    BDM_LAUNCH_CHECK("k_onco_copy");
    BDM_CUDA_TRY(cudaMemcpyAsync(out_host, c->onco_out, 2 * sizeof(long long),
                                 cudaMemcpyDeviceToHost, st));
    c->launches += 3;
    return BDM_OK;
}

}  // namespace bdm
