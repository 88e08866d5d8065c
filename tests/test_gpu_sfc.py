"""Row f1: sorting frequency and Hilbert tile order, through the C ABI.

Options "sort_every" (reorder the caller's SoA only on every K-th grid build, write
back through the input index otherwise) and "tile_order" (blocked Hilbert numbering of
the tiles) change only the memory order of the agents (R32).  The state of every agent
id after several full steps must be bit-identical to the oracle's; with sort_every the
caller's order must stay fixed between sorting builds."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _by_id(s):
    o = np.argsort(s["id"], kind="stable")
    return {k: np.asarray(v)[o] for k, v in s.items()}


def _params(orc, cfg, **over):
    from paper_2503_10796_b200 import Params
    kw = dict(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
              force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    kw.update(over)
    gp = Params(k=kw["k"], gamma=kw["gamma"], dt=kw["dt"], max_displacement=kw["max_disp"],
                force_threshold=kw["force_threshold"], detect_static=kw["detect_static"],
                collect_stats=True)
    op = orc.mech_params(k=kw["k"], gamma=kw["gamma"], dt=kw["dt"], max_disp=kw["max_disp"],
                         force_threshold=kw["force_threshold"], detect_static=kw["detect_static"])
    return gp, op


def _cluster(orc, n_bg, side_bg, n_cl, side_cl, seed):
    bg = orc.init_spheres(n_bg, seed, side_bg, 8.0, 4.0, True)
    cl = orc.init_spheres(n_cl, seed + 1, side_cl, 8.0, 4.0, True)
    off = 0.5 * (side_bg - side_cl)
    s = {k: np.concatenate([bg[k], cl[k] + off]) for k in ("x", "y", "z")}
    s["d"] = np.concatenate([bg["d"], cl["d"]])
    s["id"] = np.arange(n_bg + n_cl, dtype=np.uint32)
    s["flags"] = np.full(n_bg + n_cl, 4, np.uint32)
    return s


@pytest.mark.parametrize("mech_kernel", [0, 1, 4, 5], ids=["tile", "reference", "row", "tile7"])
@pytest.mark.parametrize("tile_order,sort_every", [(1, 1), (0, 3), (1, 0), (1, 2)])
@pytest.mark.parametrize("pop", ["cfg2", "dense", "sparse"])
def test_state_per_id_bit_exact(torch_cuda, orc, mech_kernel, tile_order, sort_every, pop):
    """sparse: about one agent per box, where the tile kernel takes two-tile units
    (auto tile depth) -- also under the Hilbert numbering."""
    from paper_2503_10796_b200 import Agents, Engine
    cfg = W.cfg2_scaled(60_000)
    if pop == "sparse":
        side = (60_000 * 1000.0 / 0.5 * 1.05) ** (1.0 / 3.0)   # d = 10, ~0.95 agents per box
        s = orc.init_spheres(60_000, 4, side, 10.0, 0.0, False)
    elif pop == "cfg2":
        s = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
        # start from an unsorted memory order (a permutation of the ids)
        perm = np.random.default_rng(3).permutation(cfg.n)
        s = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
    else:  # crowded regions: the dense-box kernel's tile list under the Hilbert numbering
        s = _cluster(orc, 20000, 220.0, 3000, 24.0, 5)
    gp, op = _params(orc, cfg)
    e = Engine(0, len(s["x"]))
    try:
        e.set_option("mech_kernel", mech_kernel)
        e.set_option("fuse_reduce", 0 if mech_kernel == 1 else 1)
        e.set_option("tile_order", tile_order)
        e.set_option("sort_every", sort_every)
        a = Agents.from_numpy(s)
        o = s
        for t in range(5):
            ids_before = a.numpy()["id"]
            e.step(a, gp, sync=True)
            st = e.stats()
            o, cnt = orc.step_full(o, op)
            g = a.numpy()
            sorting = sort_every == 1 or (sort_every > 1 and t % sort_every == 0)
            if not sorting:
                assert np.array_equal(g["id"], ids_before), f"step {t}: order changed"
            gi, oi = _by_id(g), _by_id(o)
            for k in ("id", "flags", "d", "x", "y", "z"):
                assert np.array_equal(gi[k], oi[k]), (t, k)
            assert (st["cand"], st["nbr"], st["cont"], st["n_static"]) == (
                cnt["cand"], cnt["nbr"], cnt["cont"], cnt["n_static"]), t
    finally:
        e.close()


def test_hilbert_sorted_order_follows_the_curve(torch_cuda, orc):
    """With tile_order 1 and sort_every 1 the agents after a step are ordered by the
    slot of their start-of-step box under the blocked-Hilbert numbering (then id):
    recomputed here from the grid info and the host-side curve table."""
    from paper_2503_10796_b200 import Agents, Engine, tile_curve
    cfg = W.cfg2_scaled(40_000)
    s = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    gp, _ = _params(orc, cfg)
    e = Engine(0, cfg.n)
    try:
        e.set_option("tile_order", 1)
        a = Agents.from_numpy(s)
        e.grid_build(a, gp.radius)
        gi = e.grid_info()
        e.mech_step(a, gp)
        out = a.numpy()
    finally:
        e.close()
    T = [((d + 3) // 4 + 7) // 8 * 8 for d in gi["dims"]]
    L, org = gi["L"], gi["origin"]
    h = np.asarray(tile_curve(1), np.int64)
    pos = {int(i): k for k, i in enumerate(s["id"])}
    idx = np.array([pos[int(i)] for i in out["id"]])
    b = [np.floor((s[c][idx] - org[j]) / L).astype(np.int64) for j, c in enumerate("xyz")]
    t = [v >> 2 for v in b]
    sup = ((t[2] >> 3) * (T[1] >> 3) + (t[1] >> 3)) * (T[0] >> 3) + (t[0] >> 3)
    rank = sup * 512 + h[((t[2] & 7) << 6) | ((t[1] & 7) << 3) | (t[0] & 7)]
    m = ((b[0] & 1) | ((b[1] & 1) << 1) | ((b[2] & 1) << 2) | ((b[0] & 2) << 2) |
         ((b[1] & 2) << 3) | ((b[2] & 2) << 4))
    key = rank * 64 + m
    order = np.lexsort((out["id"], key))
    assert np.array_equal(order, np.arange(cfg.n))


@pytest.mark.parametrize("inplace", [True, False])
def test_step_host_keep_order(torch_cuda, orc, inplace):
    """bdm_step_host with sort_every = 0: the host arrays keep their order; in place only
    x, y, z, flags travel back (d, id unchanged by a mechanics step), otherwise all six.
    The state per id equals the oracle's after every step."""
    import torch
    from paper_2503_10796_b200 import Agents, Engine
    cfg = W.cfg2_scaled(40_000)
    s = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    gp, op = _params(orc, cfg)
    e = Engine(0, cfg.n)
    try:
        e.set_option("sort_every", 0)
        hin = Agents.empty(cfg.n, pin=True)
        hout = Agents.empty(cfg.n, pin=True)
        for k, src in (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "d")):
            getattr(hin, k).copy_(torch.from_numpy(np.ascontiguousarray(s[src])))
        hin.id.copy_(torch.from_numpy(s["id"].view(np.int32)))
        hin.flags.copy_(torch.from_numpy(s["flags"].view(np.int32)))
        hin.n = cfg.n
        dev = Agents.empty(cfg.n)
        o = s
        src_buf = hin
        for t in range(3):
            dst = src_buf if inplace else (hout if src_buf is hin else hin)
            e.step_host(src_buf, dst, dev, gp)
            o, _ = orc.step_full(o, op)
            got = {"x": dst.x.numpy().copy(), "y": dst.y.numpy().copy(), "z": dst.z.numpy().copy(),
                   "d": dst.diameter.numpy().copy(), "id": dst.id.numpy().view(np.uint32).copy(),
                   "flags": dst.flags.numpy().view(np.uint32).copy()}
            assert np.array_equal(got["id"], s["id"]), t          # input order kept
            gi, oi = _by_id(got), _by_id(o)
            for k in ("id", "flags", "d", "x", "y", "z"):
                assert np.array_equal(gi[k], oi[k]), (t, k)
            src_buf = dst
    finally:
        e.close()
