"""GPU parity for the SIR step (cfg4) through the C ABI."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    e = Engine(0, 1 << 16)
    yield e
    e.close()


def gpu_sir_agents(eng, n, side, n_infected, seed=1, with_id=True):
    from paper_2503_10796_b200 import Agents
    a = Agents.empty(n, state=True)
    eng.init_spheres(a, n, seed=seed, side=side, d_lo=0.0)
    a.state[:n_infected] = 1
    if not with_id:
        a.id = None
    return a


def compare(a, o):
    g = a.numpy()
    for k in ("x", "y", "z", "state"):
        assert np.array_equal(g[k], o[k]), k


@pytest.mark.parametrize("n,side,n_inf,p_inf,p_rec", [
    (1, 10.0, 1, 0.1, 0.01),
    (5000, 40.0, 500, 0.3, 0.05),        # dense: many infections per step
    (20011, 60.0, 2000, 0.1, 0.01),
    (3000, 8.0, 300, 1.0, 0.0),          # D = 4 boxes per axis: heavy periodic wrap
])
def test_sir_reduced_trajectory(eng, orc, n, side, n_inf, p_inf, p_rec):
    from paper_2503_10796_b200 import Params
    a = gpu_sir_agents(eng, n, side, n_inf)
    o = orc.init_sir(n, 1, side, n_inf)
    compare(a, o)
    for t in range(8):
        counts = eng.sir_step(a, Params(seed=1, step=t), side, 2.0, p_inf, p_rec)
        o, oc, ni = orc.sir_step(o, side, 2.0, p_inf, p_rec, 1, t)
        compare(a, o)
        assert counts[:3] == list(oc) and counts[3] == ni, (t, counts, oc, ni)


def test_sir_null_ids_equal_index(eng, orc):
    from paper_2503_10796_b200 import Params
    n, side = 4000, 30.0
    a = gpu_sir_agents(eng, n, side, 400, with_id=False)
    o = orc.init_sir(n, 1, side, 400)
    for t in range(3):
        eng.sir_step(a, Params(seed=1, step=t), side, 2.0, 0.5, 0.1)
        o, _, _ = orc.sir_step(o, side, 2.0, 0.5, 0.1, 1, t)
        compare(a, o)


def test_sir_index_capacity_error(eng, orc):
    from paper_2503_10796_b200 import BdmError, Engine, Params
    e = Engine(0, 16)
    e.set_option("sir_index_capacity", 100)
    e._sir_autogrow = False
    a = gpu_sir_agents(e, 5000, 40.0, 500)
    before = a.numpy()
    with pytest.raises(BdmError) as ei:
        e.sir_step(a, Params(seed=1, step=0), 40.0, 2.0, 0.1, 0.01)
    assert ei.value.status == -2
    after = a.numpy()
    for k in ("x", "y", "z", "state"):
        assert np.array_equal(before[k], after[k])
    # with auto-grow the binding enlarges the index and re-issues the step
    e._sir_autogrow = True
    counts = e.sir_step(a, Params(seed=1, step=0), 40.0, 2.0, 0.1, 0.01)
    o, oc, _ = orc.sir_step(orc.init_sir(5000, 1, 40.0, 500), 40.0, 2.0, 0.1, 0.01, 1, 0)
    compare(a, o)
    assert counts[:3] == list(oc)
    e.close()


@pytest.mark.slow
def test_cfg4_full_size_sampled(eng, orc):
    """configs[3] at full size (100M agents, 10 km periodic cube, 0.1 % infected): two
    steps; 200k sampled agents (plus every agent whose state changed) recomputed by the
    oracle from the GPU's input snapshot must match bit-exactly; S+I+R = N."""
    import torch
    from paper_2503_10796_b200 import Params
    cfg = W.CFG4
    a = gpu_sir_agents(eng, cfg.n, cfg.side, cfg.n_infected)
    rng = np.random.default_rng(0)
    for t in range(2):
        before = a.numpy()
        counts = eng.sir_step(a, Params(seed=cfg.seed, step=t), cfg.side, cfg.radius,
                              cfg.p_inf, cfg.p_rec)
        assert sum(counts[:3]) == cfg.n
        after = a.numpy()
        changed = np.nonzero(after["state"] != before["state"])[0]
        sample = np.unique(np.concatenate([rng.choice(cfg.n, 200_000, replace=False), changed]))
        before["id"] = np.arange(cfg.n, dtype=np.uint32)
        out, _, _ = orc.sir_step_sample(before, cfg.side, cfg.radius, cfg.p_inf, cfg.p_rec,
                                        cfg.seed, t, sample)
        for k in ("x", "y", "z", "state"):
            assert np.array_equal(after[k][sample], out[k]), (t, k)
        assert counts[3] == int(np.count_nonzero((before["state"] == 0) & (after["state"] != 0)))
        del before, after
        torch.cuda.empty_cache()


def test_shared_reciprocal_division_is_ieee(eng):
    """The capped step divides the three components of v by |v| through one reciprocal
    (kernels_sir.cu div_by_recip); it must equal IEEE division bit for bit.  2^28 random
    operands of the step's range (v = 2u - 1, |v| > 1), two seeds."""
    for seed in (1, 0x9E3779B97F4A7C15):
        assert eng.selftest_recip_div(1 << 28, seed) == 0
