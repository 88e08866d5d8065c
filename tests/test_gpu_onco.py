"""GPU parity for the oncology behaviour with agent removal through the
C ABI, against the pinned oracle (tests/test_oracle_onco.py): several full steps
(mechanics with Table 4.2's adherence as the force threshold and its maximum speed as
the cap, then Alg. 4 + removal), bit-exact state incl. order, ids and ages."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    e = Engine(0, 1 << 12)
    yield e
    e.close()


def _population(orc, n, side, seed):
    s = orc.init_spheres(n, seed, side, 10.0, 4.0, True)
    s["vol"] = (math.pi / 6.0) * (s["d"] * s["d"] * s["d"])
    s["age"] = orc.init_ages(s["id"], seed, 120)
    return s


def _gpu_state(a, age_t):
    g = a.numpy()
    g["age"] = age_t.cpu().numpy().view(np.uint32)[g["id"]]
    return g


def _compare(g, o, what):
    for k in ("id", "flags", "age"):
        assert np.array_equal(g[k], o[k]), (what, k)
    for k in ("x", "y", "z", "d", "vol"):
        assert np.array_equal(g[k], o[k]), (what, k)


@pytest.mark.parametrize("n,side,p_death,p_div,steps", [
    (1, 50.0, 0.033, 0.0215, 3),
    (4000, 140.0, 0.033, 0.0215, 5),      # Table 4.2 values
    (3000, 120.0, 0.3, 0.5, 5),           # frequent removals and divisions
])
def test_onco_steps_bit_exact(eng, orc, n, side, p_death, p_div, steps):
    import torch
    from paper_2503_10796_b200 import Agents, COncoParams, Params
    s = _population(orc, n, side, 3)
    a = Agents.from_numpy(s, capacity=4 * n + 16)
    age = torch.zeros(8 * n + 64, dtype=torch.int32, device="cuda")
    age[:n].copy_(torch.from_numpy(s["age"].view(np.int32)))
    gp = Params(k=2.0, gamma=1.0, dt=1.0, max_displacement=1.0, force_threshold=1.8)
    op = orc.mech_params(k=2.0, gamma=1.0, dt=1.0, max_disp=1.0, force_threshold=1.8)
    id_next_g = id_next_o = n
    for t in range(steps):
        po = orc.onco_params(p_death=p_death, p_div=p_div, step=t, seed=7)
        pg = COncoParams.make(p_death=p_death, p_div=p_div, step=t, seed=7)
        eng.step(a, gp, sync=True)
        id_next_g = eng.onco_step(a, age, pg, id_next_g)
        s, _, id_next_o = orc.onco_full_step(s, op, po, id_next_o)
        assert id_next_g == id_next_o and a.n == len(s["x"]), t
        _compare(_gpu_state(a, age), s, f"step {t}")


def test_onco_capacity_error_leaves_state(eng, orc):
    import torch
    from paper_2503_10796_b200 import Agents, BdmError, COncoParams
    n = 500
    s = _population(orc, n, 80.0, 5)
    s["d"] = np.full(n, 14.0)
    s["vol"] = (math.pi / 6.0) * (s["d"] * s["d"] * s["d"])
    a = Agents.from_numpy(s, capacity=n + 10)            # room for 10 daughters only
    age = torch.zeros(4 * n, dtype=torch.int32, device="cuda")
    before = a.numpy()
    with pytest.raises(BdmError):
        eng.onco_step(a, age, COncoParams.make(p_div=1.0, p_death=0.0), n)
    after = a.numpy()
    for k in before:
        assert np.array_equal(before[k], after[k]), k
    assert a.n == n
