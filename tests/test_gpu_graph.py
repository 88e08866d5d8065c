"""A step captured once as a CUDA graph and replayed (bench.py's `graph` figure) gives the
same state as the same steps launched directly, and the oracle's.

Every value a replay depends on must come from device memory (the captured kernel
arguments are frozen): the grid geometry, the fused extent, the tile counters and the
slot scan's look-back tags are all device-side."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _graph_replays(eng, a, params, stream, k):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        g.capture_begin(capture_error_mode="relaxed")
        eng.grid_build(a, params.radius, stream=stream)
        eng.mech_step(a, params, stream=stream)
        g.capture_end()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(k):
            g.replay()
    torch.cuda.synchronize()
    assert eng.try_sync(stream) == 0


@pytest.mark.parametrize("n,kernel", [(50_000, 5), (50_000, 0), (3_000, 5)])
def test_graph_replay_matches_direct_and_oracle(orc, n, kernel):
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    cfg = W.cfg2_scaled(n)
    s = orc.init_spheres(n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    detect_static=True)
    op = orc.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                         detect_static=True)
    stream = torch.cuda.Stream()  # (graphs are captured on a non-default stream)
    engines = []
    for _ in range(2):
        e = Engine(0, n)
        e.set_option("mech_kernel", kernel)
        engines.append(e)
    direct, replayed = Agents.from_numpy(s), Agents.from_numpy(s)
    steps = 5
    for _ in range(steps):
        engines[0].step(direct, params, stream=stream, sync=True)
    engines[1].step(replayed, params, stream=stream, sync=True)  # sizes the grid, fused extent
    _graph_replays(engines[1], replayed, params, stream, steps - 1)
    g_d, g_r = direct.numpy(), replayed.numpy()
    for key in ("id", "flags", "d", "x", "y", "z"):
        assert np.array_equal(g_d[key], g_r[key]), key
    o = s
    for _ in range(steps):
        o, _ = orc.step_full(o, op)
    for key in ("id", "flags", "d", "x", "y", "z"):
        assert np.array_equal(g_d[key], o[key]), key
    for e in engines:
        e.close()
