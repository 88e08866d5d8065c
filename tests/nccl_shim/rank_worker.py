"""One rank of tests/test_gpu_nccl_shim.py: python rank_worker.py RANK NRANKS N STEPS OUT.
Runs the x-slab step through bdm_dist_init / bdm_aura_exchange (the NCCL code path of
dist_abi.cu, with BDM_NCCL_LIB pointing at the file-based stand-in) on its slab of a
cfg2-like cube and saves its final agents."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402


def main():
    rank, nranks, n, steps, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    from paper_2503_10796_b200.slabs import NativeSlabDomain, slab_bounds
    cfg = W.cfg2_scaled(n)
    params = Params(detect_static=True, dt=0.5)   # dt 0.5: a few agents migrate each step
    full = Agents.empty(cfg.n)
    e0 = Engine(0, cfg.n)
    e0.init_spheres(full, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                    d_random=cfg.d_random)
    torch.cuda.synchronize()
    lo, hi = slab_bounds(rank, nranks, cfg.side)
    m = (full.x[:cfg.n] >= lo) & (full.x[:cfg.n] < hi)
    k = int(m.sum())
    a = Agents.empty(k + 64)                       # small headroom: exercises the capacity path
    for f in ("x", "y", "z", "diameter", "id", "flags"):
        getattr(a, f)[:k].copy_(getattr(full, f)[:cfg.n][m])
    a.n = k
    e0.close()
    eng = Engine(0, a.capacity)
    # every rank uses the same 128 bytes (the stand-in ignores them; with NCCL rank 0's id
    # is broadcast by the caller)
    dom = NativeSlabDomain([eng], [a], [(lo, hi)], params, uid=b"shim" + bytes(124), rank=rank,
                           nranks=nranks, ghost_capacity=16)
    ghosts = []
    for _ in range(steps):
        ghosts.append(dom.step()["ghosts"])
    dom.check()
    s = a.numpy()
    np.savez(out, ghosts=np.asarray(ghosts), **{f: s[f] for f in ("x", "y", "z", "d", "id", "flags")})


if __name__ == "__main__":
    main()
