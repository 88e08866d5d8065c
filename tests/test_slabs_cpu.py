"""The x-slab protocol on the CPU: partition transparency.

A G-slab run (migration + global frame all-reduce + aura + step on locals and ghosts)
must give, agent by agent, bit-identical results to the undivided oracle run
(SURVEY 8(c3) "Partition": mirrors TeraAgent's replication of BioDynaMo).
The device side is the CPU test double tests/slab_oracle_ops.py; the protocol and the
transports are the product's paper_2503_10796_b200/slabs.py.  Two flavours: several
slabs in one process (LocalTransport) and world_size-2 gloo (DistTransport).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

N, SIDE, STEPS = 1500, 90.0, 6


def _reference(orc, steps, detect_static=False, tau=0.0):
    s = orc.init_spheres(N, 3, SIDE, 8.0, 4.0, True)
    p = orc.mech_params(detect_static=detect_static, force_threshold=tau)
    for _ in range(steps):
        out, _ = orc.mech_step(s, p)
        s = dict(s, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])
    return s


def _by_id(s):
    o = np.argsort(s["id"])
    return {k: np.asarray(v)[o] for k, v in s.items()}


def _run_slabs(G, slabs_owned, transport_factory, detect_static=False, tau=0.0, codec=False):
    import oracle
    from paper_2503_10796_b200 import Params
    from paper_2503_10796_b200.slabs import Slab, SlabDomain, slab_bounds
    from slab_oracle_ops import NpAgents, OracleOps

    s = oracle.init_spheres(N, 3, SIDE, 8.0, 4.0, True)
    op = oracle.mech_params(detect_static=detect_static, force_threshold=tau)
    slabs = []
    for g in slabs_owned:
        lo, hi = slab_bounds(g, G, SIDE)
        ops = OracleOps(op)
        agents = NpAgents.from_state(s, (s["x"] >= lo) & (s["x"] < hi))
        slabs.append(Slab(g, lo, hi, ops, agents))
    tr = transport_factory(slabs)
    dom = SlabDomain(slabs, tr, Params(detect_static=detect_static, force_threshold=tau),
                     aura_codec=codec, ref_every=3)
    stats = []
    for _ in range(STEPS):
        stats.append(dom.step())
    return {sl.g: sl.agents.state() for sl in slabs}, stats


@pytest.mark.parametrize("G,codec", [(2, False), (3, False), (5, False), (3, True)])
def test_virtual_slabs_match_undivided_run(orc, G, codec):
    """codec: the aura travels as delta + LZ4 streams (row f3), references refreshed
    every 3 iterations."""
    from paper_2503_10796_b200.slabs import LocalTransport
    ref = _by_id(_reference(orc, STEPS))
    parts, stats = _run_slabs(G, range(G), lambda slabs: LocalTransport(), codec=codec)
    got = {k: np.concatenate([parts[g][k] for g in range(G)]) for k in ref}
    got = _by_id(got)
    assert np.array_equal(got["id"], ref["id"])          # every agent exactly once
    for k in ("x", "y", "z", "flags", "d"):
        assert np.array_equal(got[k], ref[k]), k
    assert sum(st["ghosts"] for st in stats) > 0
    assert sum(st["migrated"] for st in stats) > 0       # migration actually exercised
    if codec:  # steps after the first reference travel as deltas
        assert sum(st["aura_stream_bytes"] for st in stats[1:]) < sum(
            st["aura_raw_bytes"] for st in stats[1:])


def test_virtual_slabs_static_skip(orc):
    from paper_2503_10796_b200.slabs import LocalTransport
    ref = _by_id(_reference(orc, STEPS, detect_static=True, tau=0.05))
    parts, _ = _run_slabs(3, range(3), lambda slabs: LocalTransport(), True, 0.05)
    got = _by_id({k: np.concatenate([parts[g][k] for g in range(3)]) for k in ref})
    for k in ("id", "x", "y", "z", "flags"):
        assert np.array_equal(got[k], ref[k]), k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, codec=False):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2503_10796_b200.slabs import DistTransport
    try:
        parts, stats = _run_slabs(world, [rank],
                                  lambda slabs: DistTransport(slabs[0].ops, "cpu"), codec=codec)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **parts[rank],
                 migrated=np.array([st["migrated"] for st in stats]),
                 ghosts=np.array([st["ghosts"] for st in stats]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("codec", [False, True], ids=["raw_aura", "delta_lz4_aura"])
def test_gloo_world_size_2_matches_undivided_run(orc, tmp_path, codec):
    """world_size-2 gloo run of the protocol with the DistTransport (the transport used
    over NCCL on GPUs) is bit-identical to the undivided run, with the aura sent as
    SoA fields or as delta + LZ4 byte streams (row f3)."""
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path), codec), nprocs=world,
                       join=True, start_method="spawn")
    ref = _by_id(_reference(orc, STEPS))
    parts = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    got = _by_id({k: np.concatenate([p[k] for p in parts]) for k in ref})
    for k in ("id", "x", "y", "z", "flags", "d"):
        assert np.array_equal(got[k], ref[k]), k
    assert parts[0]["ghosts"].sum() > 0 and parts[0]["migrated"].sum() + parts[1]["migrated"].sum() > 0
