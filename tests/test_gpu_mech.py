"""GPU parity: libbdm.so (through the C ABI) against the CPU oracle, same seeded inputs.

Bar (BASELINE.json north_star): neighbour pair sets, ids, order and flags bit-exact;
fp64 positions within 1e-9 relative -- the canonical summation order and fma sites
(R9) make them bit-exact, which is what these tests assert first.
"""
import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9  # north_star tolerance for fp64 positions


@pytest.fixture(scope="module", params=[(0, 1), (1, 1), (2, 1), (3, 1), (0, 2), (0, 0), (4, 0),
                                        (5, 1), (5, 2), (5, 3)],
                ids=["tile", "reference", "tile_v1", "tile_4cta", "tile_depth2", "tile_auto", "row",
                     "tile7", "tile7_depth2", "tile7_big"])
def eng(request):
    """Every mechanics kernel: the tile kernel (default; also with two-tile work units,
    option tile_depth 2, and the 8-warp two-tile units of dense populations, tile_depth 3),
    the per-agent reference and the other tile variants."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    kernel, depth = request.param
    e = Engine(0, 1 << 16)
    e.set_option("mech_kernel", kernel)
    e.set_option("tile_depth", depth)
    e.set_option("fuse_reduce", 0 if kernel == 1 else 1)  # tile kernels: fused a1
    yield e
    e.close()


def gpu_init(eng, cfg, n=None, capacity=None):
    from paper_2503_10796_b200 import Agents
    n = cfg.n if n is None else n
    a = Agents.empty(max(capacity or n, 1))
    eng.init_spheres(a, n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                     d_random=cfg.d_random)
    return a


def orc_init(orc, cfg, n=None):
    n = cfg.n if n is None else n
    return orc.init_spheres(n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)


def params_pair(orc, cfg, **over):
    from paper_2503_10796_b200 import Params
    kw = dict(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
              force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    kw.update(over)
    gp = Params(k=kw["k"], gamma=kw["gamma"], dt=kw["dt"], max_displacement=kw["max_disp"],
                force_threshold=kw["force_threshold"], detect_static=kw["detect_static"],
                boundary=kw.get("boundary", 0), lo=kw.get("lo", (0, 0, 0)),
                hi=kw.get("hi", (0, 0, 0)), collect_stats=kw.get("stats", True))
    op = orc.mech_params(k=kw["k"], gamma=kw["gamma"], dt=kw["dt"], max_disp=kw["max_disp"],
                         force_threshold=kw["force_threshold"],
                         detect_static=kw["detect_static"], boundary=kw.get("boundary", 0),
                         lo=kw.get("lo", (0, 0, 0)), hi=kw.get("hi", (0, 0, 0)))
    return gp, op


def assert_state_equal(g, o, what=""):
    """g: GPU state (sorted order), o: oracle state (oracle's sorted order)."""
    assert np.array_equal(g["id"], o["id"]), f"{what}: agent order/ids differ"
    assert np.array_equal(g["flags"], o["flags"]), f"{what}: flags differ"
    assert np.array_equal(g["d"], o["d"]), f"{what}: diameters differ"
    for k in ("x", "y", "z"):
        if not np.array_equal(g[k], o[k]):
            rel = np.abs(g[k] - o[k]) / np.maximum(np.abs(o[k]), 1e-300)
            assert rel.max() <= REL_TOL, f"{what}: {k} rel err {rel.max()}"
            pytest.fail(f"{what}: {k} not bit-exact (max rel {rel.max():.3g}, within 1e-9)")


def test_init_bit_exact_vs_oracle(eng, orc):
    for cfg, n in ((W.CFG1, 4096), (W.CFG2, 100_003)):
        a = gpu_init(eng, cfg, n)
        g = a.numpy()
        o = orc_init(orc, cfg, n)
        for k in ("x", "y", "z", "d", "id", "flags"):
            assert np.array_equal(g[k], o[k]), (cfg.name, k)


def test_cfg1_trajectory_bit_exact(eng, orc):
    """configs[0]: 4,096 agents, 10 steps, full state after every step."""
    cfg = W.CFG1
    a = gpu_init(eng, cfg)
    o = orc_init(orc, cfg)
    gp, op = params_pair(orc, cfg)
    for t in range(cfg.steps):
        eng.step(a, gp, sync=True)
        st = eng.stats()
        o, cnt = orc.step_full(o, op)
        assert_state_equal(a.numpy(), o, f"cfg1 step {t}")
        for k in ("cand", "nbr", "cont", "n_static"):
            assert st[k] == cnt[k], (t, k, st[k], cnt[k])


def test_neighbor_pairs_equal_bruteforce(eng, orc):
    from paper_2503_10796_b200 import Agents
    cfg = W.CFG1
    o = orc_init(orc, cfg)
    for t in range(3):
        a = Agents.from_numpy(o)
        got = eng.neighbor_pairs(a)
        want = orc.neighbor_pairs_brute(o, float(o["d"].max()))
        assert np.array_equal(got, want)
        o, _ = orc.step_full(o, orc.mech_params())
    # ragged sizes, several densities, explicit radius
    for n, side, R in ((1, 10.0, 0.0), (2, 5.0, 0.0), (777, 60.0, 0.0), (5000, 90.0, 7.5)):
        s = orc.init_spheres(n, 3, side, 8.0, 4.0, True)
        a = Agents.from_numpy(s)
        got = eng.neighbor_pairs(a, R)
        want = orc.neighbor_pairs_brute(s, R if R > 0 else float(s["d"].max()))
        assert np.array_equal(got, want), n


@pytest.mark.parametrize("n", [1, 2, 31, 257, 20_011])
def test_cfg2_mix_reduced_n_static_on(eng, orc, n):
    """cfg2 density and diameter mix at reduced N (spans many tiles + a ragged tail)."""
    cfg = W.cfg2_scaled(n)
    a = gpu_init(eng, cfg)
    o = orc_init(orc, cfg)
    gp, op = params_pair(orc, cfg)
    for t in range(4):
        eng.step(a, gp, sync=True)
        st = eng.stats()
        o, cnt = orc.step_full(o, op)
        assert_state_equal(a.numpy(), o, f"n={n} step {t}")
        assert (st["cand"], st["nbr"], st["cont"], st["n_static"]) == (
            cnt["cand"], cnt["nbr"], cnt["cont"], cnt["n_static"])


@pytest.mark.parametrize("side,tau", [(160.0, 1e-3), (640.0, 0.0)])
def test_static_skip_fires_and_matches_oracle(eng, orc, side, tau):
    """Static skip on: bit-exact vs the oracle, and transparent vs skip off."""
    cfg = W.CFG1
    a_on = gpu_init(eng, cfg)
    eng.init_spheres(a_on, cfg.n, seed=1, side=side, d_lo=10.0)
    a_off = gpu_init(eng, cfg)
    eng.init_spheres(a_off, cfg.n, seed=1, side=side, d_lo=10.0)
    o = orc.init_spheres(cfg.n, 1, side, 10.0)
    gp_on, op_on = params_pair(orc, cfg, detect_static=True, force_threshold=tau)
    gp_off, _ = params_pair(orc, cfg, detect_static=False, force_threshold=tau)
    n_static = 0
    for t in range(8):
        eng.step(a_on, gp_on, sync=True)
        n_static += eng.stats()["n_static"]
        eng.step(a_off, gp_off, sync=True)
        o, _ = orc.step_full(o, op_on)
        g_on = a_on.numpy()
        assert_state_equal(g_on, o, f"static on step {t}")
        g_off = a_off.numpy()
        assert np.array_equal(g_on["id"], g_off["id"])
        for k in ("x", "y", "z"):
            assert np.array_equal(g_on[k], g_off[k])
    assert n_static > 100


def test_edge_cases(eng, orc):
    from paper_2503_10796_b200 import Agents, Params
    # n = 0: valid no-op
    a = Agents.empty(4)
    a.n = 0
    eng.step(a, Params(), sync=True)
    # all agents in one box; coincident centres (dist = 0 contributes nothing, R10)
    s = {"x": np.array([1.0, 1.0, 1.5, 2.0]), "y": np.array([0.0, 0.0, 0.5, 0.25]),
         "z": np.zeros(4), "d": np.full(4, 10.0), "id": np.arange(4, dtype=np.uint32),
         "flags": np.full(4, 4, np.uint32)}
    a = Agents.from_numpy(s)
    gp, op = params_pair(orc, W.CFG1)
    eng.step(a, gp, sync=True)
    o, _ = orc.step_full(s, op)
    assert_state_equal(a.numpy(), o, "one box")
    # heavy overlap with a large dt: the 3 um cap binds (R6)
    s = orc.init_spheres(3000, 2, 40.0, 10.0)
    a = Agents.from_numpy(s)
    gp, op = params_pair(orc, W.CFG1, dt=1.0)
    eng.step(a, gp, sync=True)
    o, _ = orc.step_full(s, op)
    assert_state_equal(a.numpy(), o, "cap")
    # closed boundary (clamp into [lo, hi])
    s = orc.init_spheres(2000, 4, 50.0, 10.0)
    a = Agents.from_numpy(s)
    gp, op = params_pair(orc, W.CFG1, dt=1.0, boundary=1, lo=(5, 5, 5), hi=(45, 45, 45))
    eng.step(a, gp, sync=True)
    o, _ = orc.step_full(s, op)
    assert_state_equal(a.numpy(), o, "closed")


@pytest.mark.parametrize("k", [23, 24, 25, 40, 90])
def test_crowded_neighbourhoods(eng, orc, k):
    """An agent with exactly k agents inside its radius (around the per-agent list
    capacity of the tile kernel and beyond): bit-exact vs the oracle."""
    from paper_2503_10796_b200 import Agents
    rng = np.random.default_rng(k)
    # k neighbours inside a ball of radius 9 (R = 10) around the origin + sparse others
    v = rng.normal(size=(k, 3))
    v *= (rng.uniform(0.2, 0.9, k) ** (1 / 3) * 9.0 / np.linalg.norm(v, axis=1))[:, None]
    far = rng.uniform(-60, 60, (300, 3))
    pts = np.vstack([[0, 0, 0], v, far])
    n = len(pts)
    s = {"x": pts[:, 0].copy(), "y": pts[:, 1].copy(), "z": pts[:, 2].copy(),
         "d": np.full(n, 10.0), "id": np.arange(n, dtype=np.uint32),
         "flags": np.full(n, 4, np.uint32)}
    gp, op = params_pair(orc, W.CFG1)
    a = Agents.from_numpy(s)
    for t in range(2):
        eng.step(a, gp, sync=True)
        s, _ = orc.step_full(s, op)
        assert_state_equal(a.numpy(), s, f"k={k} step {t}")


def _dense_population(orc, n_bg, side_bg, n_cl, side_cl, seed):
    """A uniform background (n_bg agents, cfg2 diameter mix, cube side_bg) plus a dense
    cluster of n_cl agents in a cube of side side_cl at its centre (ids follow on)."""
    bg = orc.init_spheres(n_bg, seed, side_bg, 8.0, 4.0, True)
    cl = orc.init_spheres(n_cl, seed + 1, side_cl, 8.0, 4.0, True)
    off = 0.5 * (side_bg - side_cl)
    s = {}
    for k in ("x", "y", "z"):
        s[k] = np.concatenate([bg[k], cl[k] + off])
    s["d"] = np.concatenate([bg["d"], cl["d"]])
    s["id"] = np.arange(n_bg + n_cl, dtype=np.uint32)
    s["flags"] = np.full(n_bg + n_cl, 4, np.uint32)
    return s


@pytest.mark.parametrize("n_bg,side_bg,n_cl,side_cl,static,tau", [
    (0, 1.0, 6000, 40.0, False, 0.0),        # every region dense, ~100 agents per box
    (20000, 220.0, 3000, 24.0, True, 1e-3),  # dense cluster inside sparse tiles, static on
    (4000, 120.0, 1500, 14.0, True, 0.0),    # > 32 agents per box (several lane groups)
])
def test_dense_regions(eng, orc, n_bg, side_bg, n_cl, side_cl, static, tau):
    """Regions too crowded for the tile kernel's staging (cfg3 late-step densities) go to
    the dense-box kernel: candidate streams longer than one staged batch, boxes with
    more agents than lanes, mixed with sparse tiles; bit-exact state and counters."""
    from paper_2503_10796_b200 import Agents
    s = _dense_population(orc, n_bg, side_bg, n_cl, side_cl, 5)
    gp, op = params_pair(orc, W.CFG1, detect_static=static, force_threshold=tau)
    a = Agents.from_numpy(s)
    for t in range(3):
        eng.step(a, gp, sync=True)
        st = eng.stats()
        s, cnt = orc.step_full(s, op)
        assert_state_equal(a.numpy(), s, f"dense step {t}")
        assert (st["cand"], st["nbr"], st["cont"], st["n_static"]) == (
            cnt["cand"], cnt["nbr"], cnt["cont"], cnt["n_static"]), t


def test_capacity_overflow_is_recovered(eng, orc):
    """An agent far outside the first grid's extent exceeds the slot capacity; the
    overflowed step is a no-op and the binding grows the slots and re-issues it."""
    from paper_2503_10796_b200 import Agents, Engine
    e = Engine(0, 16)
    e.set_option("mech_kernel", eng.lib and 0)
    s = orc.init_spheres(500, 5, 50.0, 10.0)
    a = Agents.from_numpy(s)
    gp, op = params_pair(orc, W.CFG1)
    e.step(a, gp, sync=True)
    s1, _ = orc.step_full(s, op)
    s1 = {k: v.copy() for k, v in s1.items()}
    s1["x"][0] += 5000.0
    a = Agents.from_numpy(s1)
    e.step(a, gp, sync=True)
    o, _ = orc.step_full(s1, op)
    assert_state_equal(a.numpy(), o, "after regrow")
    e.close()


def test_step_host_equals_device_step(eng, orc):
    import torch
    from paper_2503_10796_b200 import Agents
    cfg = W.cfg2_scaled(50_000)
    o = orc_init(orc, cfg)
    hin = Agents.empty(cfg.n, pin=True)
    hout = Agents.empty(cfg.n, pin=True)
    for k, src in (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "d")):
        getattr(hin, k).copy_(torch.from_numpy(o[src]))
    hin.id.copy_(torch.from_numpy(o["id"].view(np.int32)))
    hin.flags.copy_(torch.from_numpy(o["flags"].view(np.int32)))
    hin.n = cfg.n
    dev = Agents.empty(cfg.n)
    gp, op = params_pair(orc, cfg)
    eng.step_host(hin, hout, dev, gp)
    want, _ = orc.step_full(o, op)
    got = {"x": hout.x.numpy(), "y": hout.y.numpy(), "z": hout.z.numpy(),
           "d": hout.diameter.numpy(), "id": hout.id.numpy().view(np.uint32),
           "flags": hout.flags.numpy().view(np.uint32)}
    assert_state_equal(got, want, "step_host")


def test_step_host_new_input_ignores_fused_extent(eng, orc):
    """bdm_step_host overwrites the device arrays from the host, so a fused extent left
    by the previous step (option fuse_reduce) must not be reused: a second call with
    different host data (shifted by 40 um) still matches the oracle."""
    import torch
    from paper_2503_10796_b200 import Agents
    cfg = W.cfg2_scaled(30_000)
    gp, op = params_pair(orc, cfg)
    dev = Agents.empty(cfg.n)
    hin = Agents.empty(cfg.n, pin=True)
    hout = Agents.empty(cfg.n, pin=True)
    for shift in (0.0, 40.0):
        o = orc_init(orc, cfg)
        for k in ("x", "y", "z"):
            o[k] = o[k] + shift
        for k, src in (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "d")):
            getattr(hin, k).copy_(torch.from_numpy(o[src]))
        hin.id.copy_(torch.from_numpy(o["id"].view(np.int32)))
        hin.flags.copy_(torch.from_numpy(o["flags"].view(np.int32)))
        hin.n = cfg.n
        eng.step_host(hin, hout, dev, gp)
        want, _ = orc.step_full(o, op)
        got = {"x": hout.x.numpy(), "y": hout.y.numpy(), "z": hout.z.numpy(),
               "d": hout.diameter.numpy(), "id": hout.id.numpy().view(np.uint32),
               "flags": hout.flags.numpy().view(np.uint32)}
        assert_state_equal(got, want, f"step_host shift {shift}")


@pytest.mark.slow
def test_cfg2_full_size_teacher_forced(eng, orc):
    """configs[1] at full size (10M agents), the bench's launch configuration: after
    steps 0 and 1, 100k sampled agents recomputed by the oracle from the GPU's input
    state (teacher forcing) must match bit-exactly."""
    import torch
    cfg = W.CFG2
    a = gpu_init(eng, cfg)
    gp, op = params_pair(orc, cfg)
    rng = np.random.default_rng(0)
    for t in range(2):
        before = a.numpy()
        eng.step(a, gp, sync=True)
        after = a.numpy()
        sample = rng.choice(cfg.n, 100_000, replace=False)
        out, cnt = orc.mech_step(before, op, sample=sample)
        pos = {int(i): k for k, i in enumerate(after["id"])}
        idx = np.array([pos[int(before["id"][i])] for i in sample])
        for k in ("x", "y", "z", "flags"):
            g = after[k][idx]
            assert np.array_equal(g, out[k]), (t, k)
        # the order is the oracle's sorted order of the input state
        perm, _ = orc.sorted_order(before)
        assert np.array_equal(after["id"], before["id"][perm])
        del before, after
        torch.cuda.empty_cache()


@pytest.mark.slow
def test_cfg2_bench_instance_teacher_forced(orc):
    """The exact instance bench.py times: cfg2 at full size (10M agents), the default
    mechanics kernel, counters off (collect_stats = False) and the next step's grid
    extent fused into the mechanics epilogue (fuse_reduce = 1), three consecutive steps
    without a synchronizing check in between; after each, 100k sampled agents
    recomputed by the oracle from the GPU's input state must match bit-exactly."""
    import torch
    from paper_2503_10796_b200 import Engine, Params
    cfg = W.CFG2
    e = Engine(0, cfg.n)
    e.set_option("fuse_reduce", 1)
    a = gpu_init(e, cfg)
    gp = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    op = orc.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                         force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    rng = np.random.default_rng(1)
    for t in range(3):
        before = a.numpy()
        e.step(a, gp)                       # asynchronous, as in the timed loop
        after = a.numpy()
        sample = rng.choice(cfg.n, 100_000, replace=False)
        out, _ = orc.mech_step(before, op, sample=sample)
        pos = {int(i): k for k, i in enumerate(after["id"])}
        idx = np.array([pos[int(before["id"][i])] for i in sample])
        for k in ("x", "y", "z", "flags"):
            assert np.array_equal(after[k][idx], out[k]), (t, k)
        perm, _ = orc.sorted_order(before)
        assert np.array_equal(after["id"], before["id"][perm])
        del before, after
        torch.cuda.empty_cache()
    e.sync()
    e.close()


@pytest.mark.parametrize("case", ["cfg2@20011", "dense_all", "dense_cluster_static", "dense_groups",
                                  "crowded18", "crowded19", "crowded20", "crowded25", "crowded90",
                                  "cap"])
def test_counters_off_bit_exact(eng, orc, case):
    """The timed instances run without counters (collect_stats = 0): there the tile7 and
    dense kernels test contacts only in fp32 (r'_i + r'_j) for every lane that needs no
    more, and trim boxes at the contact reach.  Same populations as the counting tests,
    state bit-exact after every step; crowded18/19/20 put the central agent's survivor
    list (its contacts and itself) right at the tile7 walk's list capacity (20 entries:
    a list that reaches it sends the batch to the reference formulation)."""
    from paper_2503_10796_b200 import Agents
    if case.startswith("cfg2"):
        cfg = W.cfg2_scaled(20011)
        s = orc_init(orc, cfg)
        gp, op = params_pair(orc, cfg, stats=False)
    elif case.startswith("dense"):
        n_bg, side_bg, n_cl, side_cl, static, tau = {
            "dense_all": (0, 1.0, 6000, 40.0, False, 0.0),
            "dense_cluster_static": (20000, 220.0, 3000, 24.0, True, 1e-3),
            "dense_groups": (4000, 120.0, 1500, 14.0, True, 0.0)}[case]
        s = _dense_population(orc, n_bg, side_bg, n_cl, side_cl, 5)
        gp, op = params_pair(orc, W.CFG1, detect_static=static, force_threshold=tau, stats=False)
    elif case.startswith("crowded"):
        k = int(case[7:])
        rng = np.random.default_rng(k)
        v = rng.normal(size=(k, 3))
        v *= (rng.uniform(0.2, 0.9, k) ** (1 / 3) * 9.0 / np.linalg.norm(v, axis=1))[:, None]
        pts = np.vstack([[0, 0, 0], v, rng.uniform(-60, 60, (300, 3))])
        n = len(pts)
        s = {"x": pts[:, 0].copy(), "y": pts[:, 1].copy(), "z": pts[:, 2].copy(),
             "d": np.full(n, 10.0), "id": np.arange(n, dtype=np.uint32),
             "flags": np.full(n, 4, np.uint32)}
        gp, op = params_pair(orc, W.CFG1, stats=False)
    else:  # heavy overlap, large dt: the cap binds
        s = orc.init_spheres(3000, 2, 40.0, 10.0)
        gp, op = params_pair(orc, W.CFG1, dt=1.0, stats=False)
    a = Agents.from_numpy(s)
    for t in range(3):
        eng.step(a, gp, sync=True)
        s, _ = orc.step_full(s, op)
        assert_state_equal(a.numpy(), s, f"{case} step {t}")
