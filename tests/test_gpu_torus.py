"""GPU parity of the toroidal mechanics (boundary 2, reading R52) through the
C ABI (bdm_step): state bit-exact against the oracle after every step, counters equal,
for populations that fill the periodic cube (pairs across every face and edge), with
and without the static skip, and with the counters off (the plain instance)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _params(orc, side, stats, static, dt=0.01):
    from paper_2503_10796_b200 import Params
    gp = Params(k=2.0, gamma=1.0, dt=dt, max_displacement=3.0, detect_static=static, boundary=2,
                lo=(0.0, 0.0, 0.0), hi=(side, side, side), collect_stats=stats)
    op = orc.mech_params(k=2.0, gamma=1.0, dt=dt, max_disp=3.0, detect_static=static, boundary=2,
                         lo=(0.0, 0.0, 0.0), hi=(side, side, side))
    return gp, op


@pytest.fixture(scope="module")
def eng():
    from paper_2503_10796_b200 import Engine
    e = Engine(0, 1 << 16)
    yield e
    e.close()


@pytest.mark.parametrize("n,stats,static,dt", [(3000, True, False, 0.01), (20011, True, True, 0.01),
                                               (20011, False, True, 0.01), (5000, True, False, 0.5)])
def test_torus_trajectory_bit_exact(eng, orc, n, stats, static, dt):
    from paper_2503_10796_b200 import Agents
    cfg = W.cfg2_scaled(n)
    side = cfg.side
    s = orc.init_spheres(n, 3, side, 8.0, 4.0, d_random=True)
    gp, op = _params(orc, side, stats, static, dt)
    a = Agents.from_numpy(s)
    for t in range(4):
        eng.step(a, gp, sync=True)
        st = eng.stats()
        s, cnt = orc.step_full(s, op)
        g = a.numpy()
        for k in ("id", "flags", "d", "x", "y", "z"):
            assert np.array_equal(g[k], s[k]), (t, k)
        assert np.all((g["x"] >= 0.0) & (g["x"] <= side))
        if stats:
            assert (st["cand"], st["nbr"], st["cont"], st["n_static"]) == (
                cnt["cand"], cnt["nbr"], cnt["cont"], cnt["n_static"]), t


def test_torus_pair_across_face(eng, orc):
    from paper_2503_10796_b200 import Agents
    side = 100.0
    s = {"x": np.array([1.0, side - 1.0]), "y": np.array([50.0, 50.0]), "z": np.array([50.0, 50.0]),
         "d": np.array([10.0, 10.0]), "id": np.arange(2, dtype=np.uint32),
         "flags": np.full(2, 4, np.uint32)}
    gp, op = _params(orc, side, True, False)
    a = Agents.from_numpy(s)
    eng.step(a, gp, sync=True)
    o, cnt = orc.step_full(s, op)
    g = a.numpy()
    for k in ("id", "x", "y", "z", "flags"):
        assert np.array_equal(g[k], o[k]), k
    assert eng.stats()["cont"] == 2 == cnt["cont"]


def test_torus_invalid_rejected(eng, orc):
    from paper_2503_10796_b200 import Agents, BdmError
    s = orc.init_spheres(100, 1, 25.0, 10.0)
    a = Agents.from_numpy(s)
    gp, _ = _params(orc, 25.0, True, False)      # 2 boxes of edge >= 10 per axis
    with pytest.raises(BdmError):
        eng.step(a, gp, sync=True)
    from paper_2503_10796_b200 import Params
    bad = Params(boundary=2, lo=(0.0, 0.0, 0.0), hi=(100.0, 100.0, 90.0))
    with pytest.raises(BdmError):
        eng.step(a, bad, sync=True)
