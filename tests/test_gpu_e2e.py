"""The end-to-end entry points on host state: bdm_run_host (K steps, uploads of step
k+1 overlapping downloads of step k chunk by chunk) leaves exactly the host state that
K calls of bdm_step_host leave, which is the oracle's trajectory."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _host(s, n):
    import torch
    from paper_2503_10796_b200 import Agents
    h = Agents.empty(n, pin=True)
    for k, src in (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "d")):
        getattr(h, k)[:n].copy_(torch.from_numpy(np.ascontiguousarray(s[src], np.float64)))
    h.id[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["id"], np.uint32).view(np.int32)))
    h.flags[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["flags"], np.uint32).view(np.int32)))
    h.n = n
    return h


def _state(h):
    n = h.n
    return {"x": h.x[:n].numpy().copy(), "y": h.y[:n].numpy().copy(), "z": h.z[:n].numpy().copy(),
            "d": h.diameter[:n].numpy().copy(), "id": h.id[:n].numpy().view(np.uint32).copy(),
            "flags": h.flags[:n].numpy().view(np.uint32).copy()}


@pytest.mark.parametrize("n,sort_every,chunks", [(20011, 0, 8), (20011, 1, 8), (3001, 1, 3),
                                                 (50000, 0, 64), (7, 1, 5)])
def test_run_host_equals_step_host_and_oracle(orc, n, sort_every, chunks):
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    cfg = W.cfg2_scaled(n)
    s = orc.init_spheres(n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    detect_static=True)
    op = orc.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                         detect_static=True)
    steps = 4
    stream = torch.cuda.Stream()
    e1, e2 = Engine(0, n), Engine(0, n)
    for e in (e1, e2):
        e.set_option("sort_every", sort_every)
    h1, h2 = _host(s, n), _host(s, n)
    d1, d2 = Agents.empty(n), Agents.empty(n)
    for _ in range(steps):
        e1.step_host(h1, h1, d1, params, stream=stream)
    e2.run_host(h2, d2, params, steps, chunks=chunks, stream=stream)
    torch.cuda.synchronize()
    a, b = _state(h1), _state(h2)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    # the oracle: sort_every 1 leaves the grid order (as step_full); 0 keeps the input
    # order, so compare by id
    o = s
    for _ in range(steps):
        o, _ = orc.step_full(o, op)
    ia, io = np.argsort(b["id"]), np.argsort(o["id"])
    for k in ("x", "y", "z", "d", "flags"):
        assert np.array_equal(b[k][ia], o[k][io]), k
    for e in (e1, e2):
        e.close()
