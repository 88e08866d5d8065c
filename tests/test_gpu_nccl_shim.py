"""The multi-rank code path of bdm_aura_exchange (dist_abi.cu: bdm_dist_init with
nranks > 1, the all-reduced frame, the count exchange, the grouped per-field sends and
receives to the left and right neighbours, zero-size skips, the edge ranks) on ONE GPU:
the ranks are separate processes sharing the device, and BDM_NCCL_LIB points the library
at a file-based stand-in for the nine NCCL calls it uses (tests/nccl_shim/shim_nccl.cpp;
only hosts wait, no kernel waits on another rank).  What NCCL itself does is not tested
here; that the library's calls pair up, carry the right sizes and give the undivided
result is."""
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM_SRC = os.path.join(ROOT, "tests", "nccl_shim", "shim_nccl.cpp")
WORKER = os.path.join(ROOT, "tests", "nccl_shim", "rank_worker.py")


def _by_id(s):
    o = np.argsort(s["id"], kind="stable")
    return {k: np.asarray(v)[o] for k, v in s.items()}


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    so = str(tmp_path_factory.mktemp("shim") / "libshim_nccl.so")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-O1", "-shared", "-fPIC", "-I", os.path.join(cuda, "include"), SHIM_SRC, "-o", so,
                    "-L", os.path.join(cuda, "lib64"), "-lcudart"], check=True)
    return so


@pytest.mark.parametrize("nranks,n", [(2, 20_000), (3, 40_000)])
def test_ranked_exchange_bit_identical_to_undivided(shim, orc, tmp_path, nranks, n):
    steps = 5
    env = dict(os.environ, BDM_NCCL_LIB=shim, BDM_SHIM_DIR=str(tmp_path))
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(nranks)]
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(nranks), str(n), str(steps), outs[r]],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(nranks)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("a rank timed out")
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
    parts = [np.load(o) for o in outs]
    got = _by_id({k: np.concatenate([p[k] for p in parts]) for k in ("x", "y", "z", "d", "id", "flags")})
    assert all((p["ghosts"] > 0).all() for p in parts)        # every rank received an aura every step
    # the undivided GPU run
    from paper_2503_10796_b200 import Agents, Engine, Params
    cfg = W.cfg2_scaled(n)
    params = Params(detect_static=True, dt=0.5)
    a = Agents.empty(cfg.n)
    e = Engine(0, cfg.n)
    e.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                   d_random=cfg.d_random)
    for _ in range(steps):
        e.step(a, params, sync=True)
    ref = _by_id(a.numpy())
    assert np.array_equal(got["id"], ref["id"])               # every agent exactly once
    for k in ("x", "y", "z", "d", "flags"):
        assert np.array_equal(got[k], ref[k]), k
    # and the oracle
    o = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    op = orc.mech_params(detect_static=True, dt=0.5)
    for _ in range(steps):
        out, _ = orc.mech_step(o, op)
        o = dict(o, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])
    o = _by_id(o)
    for k in ("x", "y", "z", "flags"):
        assert np.array_equal(got[k], o[k]), k
    # migration happened: some agent ended on another rank than it started on
    moved = 0
    from paper_2503_10796_b200.slabs import slab_bounds
    x0 = orc.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    start = {}
    for r in range(nranks):
        lo, hi = slab_bounds(r, nranks, cfg.side)
        for i in np.asarray(x0["id"])[(np.asarray(x0["x"]) >= lo) & (np.asarray(x0["x"]) < hi)]:
            start[int(i)] = r
    for r, p in enumerate(parts):
        moved += sum(1 for i in p["id"] if start[int(i)] != r)
    assert moved > 0
