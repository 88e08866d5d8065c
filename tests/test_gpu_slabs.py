"""x-slab decomposition on the GPU, virtual-slab mode: G slabs with their
own libbdm contexts on one device, exchanging aura and migrants through the same
protocol (paper_2503_10796_b200/slabs.py) that runs over NCCL on several GPUs.
Partition transparency: bit-identical to the undivided single-context run and to the
oracle."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _by_id(s):
    o = np.argsort(s["id"])
    return {k: np.asarray(v)[o] for k, v in s.items()}


def _slab_run(G, cfg, steps, params, codec=False):
    import torch
    from paper_2503_10796_b200 import Agents, Engine
    from paper_2503_10796_b200.slabs import LibOps, LocalTransport, Slab, SlabDomain, slab_bounds
    full = Agents.empty(cfg.n)
    e0 = Engine(0, cfg.n)
    e0.init_spheres(full, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo,
                    d_width=cfg.d_width, d_random=cfg.d_random)
    torch.cuda.synchronize()
    slabs = []
    for g in range(G):
        lo, hi = slab_bounds(g, G, cfg.side)
        m = (full.x[:cfg.n] >= lo) & (full.x[:cfg.n] < hi)
        n = int(m.sum())
        a = Agents.empty(2 * cfg.n // G + 1024)
        for k in ("x", "y", "z", "diameter", "id", "flags"):
            getattr(a, k)[:n].copy_(getattr(full, k)[:cfg.n][m])
        a.n = n
        slabs.append(Slab(g, lo, hi, LibOps(Engine(0, a.capacity)), a))
    dom = SlabDomain(slabs, LocalTransport(), params, aura_codec=codec, ref_every=2)
    stats = [dom.step() for _ in range(steps)]
    torch.cuda.synchronize()
    parts = [s.agents.numpy() for s in slabs]
    got = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    return _by_id(got), stats


@pytest.mark.parametrize("G,n,codec", [(2, 20_000, False), (4, 60_000, False), (8, 100_003, False),
                                       (4, 60_000, True)])
def test_virtual_slabs_bit_identical(orc, G, n, codec):
    """codec: the aura travels as delta + LZ4 streams (row f3, bdm_aura_*), references
    refreshed every 2 iterations."""
    from paper_2503_10796_b200 import Agents, Engine, Params
    cfg = W.cfg2_scaled(n)
    params = Params(detect_static=True)
    got, stats = _slab_run(G, cfg, 4, params, codec)
    # undivided GPU run
    a = Agents.empty(cfg.n)
    e = Engine(0, cfg.n)
    e.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                   d_random=cfg.d_random)
    for _ in range(4):
        e.step(a, params, sync=True)
    ref = _by_id(a.numpy())
    assert np.array_equal(got["id"], ref["id"])
    for k in ("x", "y", "z", "d", "flags"):
        assert np.array_equal(got[k], ref[k]), k
    # and the oracle
    o = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    op = orc.mech_params(detect_static=True)
    for _ in range(4):
        out, _ = orc.mech_step(o, op)
        o = dict(o, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])
    o = _by_id(o)
    for k in ("x", "y", "z", "flags"):
        assert np.array_equal(got[k], o[k]), k
    assert sum(s["ghosts"] for s in stats) > 0
    if codec:
        assert sum(s["aura_stream_bytes"] for s in stats[1:]) < sum(
            s["aura_raw_bytes"] for s in stats[1:])


def _native_run(G, cfg, steps, params):
    import torch
    from paper_2503_10796_b200 import Agents, Engine
    from paper_2503_10796_b200.slabs import NativeSlabDomain, slab_bounds
    full = Agents.empty(cfg.n)
    e0 = Engine(0, cfg.n)
    e0.init_spheres(full, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo,
                    d_width=cfg.d_width, d_random=cfg.d_random)
    torch.cuda.synchronize()
    engines, agents, bounds = [], [], []
    for g in range(G):
        lo, hi = slab_bounds(g, G, cfg.side)
        m = (full.x[:cfg.n] >= lo) & (full.x[:cfg.n] < hi)
        n = int(m.sum())
        a = Agents.empty(n + 64)          # small headroom: exercises the capacity path
        for k in ("x", "y", "z", "diameter", "id", "flags"):
            getattr(a, k)[:n].copy_(getattr(full, k)[:cfg.n][m])
        a.n = n
        engines.append(Engine(0, a.capacity))
        agents.append(a)
        bounds.append((lo, hi))
    dom = NativeSlabDomain(engines, agents, bounds, params, ghost_capacity=16)
    stats = [dom.step() for _ in range(steps)]
    dom.check()
    parts = [a.numpy() for a in agents]
    got = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    return _by_id(got), stats


@pytest.mark.parametrize("G,n", [(1, 5_000), (2, 20_000), (4, 60_000), (8, 100_003)])
def test_native_exchange_bit_identical(orc, G, n):
    """The C-ABI exchange (bdm_dist_init_virtual / bdm_aura_exchange_virtual: frame,
    migration and aura in one call, the one-round protocol) is partition-transparent:
    bit-identical to the undivided GPU run and the oracle after 5 steps, no agent lost
    or duplicated, capacity shortfalls (tiny ghost buffers, tight local arrays) grown
    and completed."""
    from paper_2503_10796_b200 import Agents, Engine, Params
    cfg = W.cfg2_scaled(n)
    params = Params(detect_static=True, dt=0.5)   # dt 0.5: a few agents migrate each step
    got, stats = _native_run(G, cfg, 5, params)
    a = Agents.empty(cfg.n)
    e = Engine(0, cfg.n)
    e.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                   d_random=cfg.d_random)
    for _ in range(5):
        e.step(a, params, sync=True)
    ref = _by_id(a.numpy())
    assert np.array_equal(got["id"], ref["id"])   # every agent exactly once
    for k in ("x", "y", "z", "d", "flags"):
        assert np.array_equal(got[k], ref[k]), k
    o = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    op = orc.mech_params(detect_static=True, dt=0.5)
    for _ in range(5):
        out, _ = orc.mech_step(o, op)
        o = dict(o, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])
    o = _by_id(o)
    for k in ("x", "y", "z", "flags"):
        assert np.array_equal(got[k], o[k]), k
    if G > 1:
        assert all(s["ghosts"] > 0 for s in stats)


def test_pack_slab_and_append(eng=None):
    """Device packing: order-preserving selection, migration compaction, capacity error."""
    import torch
    from paper_2503_10796_b200 import Agents, BdmError, Engine
    from paper_2503_10796_b200.bdm import PACK_AURA, PACK_MIGRATE
    e = Engine(0, 1000)
    a = Agents.empty(1000)
    e.init_spheres(a, 1000, seed=2, side=100.0, d_lo=10.0)
    before = a.numpy()
    L, R = Agents.empty(1000), Agents.empty(1000)
    nl, nr = e.pack_slab(a, 30.0, 70.0, 5.0, PACK_AURA, L, R)
    x = before["x"]
    # the send buffers hold exactly the selected agents (in no particular order)
    assert np.array_equal(np.sort(L.numpy()["id"]), np.sort(before["id"][x < 35.0]))
    assert np.array_equal(np.sort(R.numpy()["id"]), np.sort(before["id"][x >= 65.0]))
    gl = L.numpy()
    pos = {int(i): k for k, i in enumerate(before["id"])}
    for k in ("x", "y", "z", "d", "flags"):
        assert np.array_equal(gl[k], before[k][[pos[int(i)] for i in gl["id"]]]), k
    assert a.n == 1000
    nl, nr = e.pack_slab(a, 30.0, 70.0, 0.0, PACK_MIGRATE, L, R)
    keep = (x >= 30.0) & (x < 70.0)
    assert a.n == int(keep.sum())
    after = a.numpy()
    # the remaining agents are the stayers (the last ones moved into the leavers' slots)
    o_after, o_want = np.argsort(after["id"]), np.argsort(before["id"][keep])
    for k in ("x", "y", "z", "d", "id", "flags"):
        assert np.array_equal(after[k][o_after], before[k][keep][o_want]), k
    stay_below = keep[:a.n]
    assert np.array_equal(after["id"][:a.n][stay_below], before["id"][:a.n][stay_below])
    assert np.array_equal(np.sort(L.numpy()["x"]), np.sort(x[x < 30.0]))
    e.append(a, L)
    assert a.n == int(keep.sum()) + nl
    small = Agents.empty(5)
    with pytest.raises(BdmError):
        e.pack_slab(a, 30.0, 70.0, 0.0, PACK_MIGRATE, small, small)
    assert a.n == int(keep.sum()) + nl            # untouched
    frame = torch.empty(4, dtype=torch.float64, device="cuda")
    e.local_frame(a, frame)
    f = frame.cpu().numpy()
    s = a.numpy()
    assert f[0] == s["x"].min() and f[1] == s["y"].min() and f[3] == -s["d"].max()
