"""bdm_create_ex: the workspace taken from the caller's allocator (torch's
caching allocator through ctypes callbacks) and sized for locals + ghosts.  The result
must not depend on where the workspace lives: the trajectory stays bit-exact against the
oracle, growth goes through the callbacks, and bdm_destroy returns every block."""
import ctypes

import numpy as np
import pytest

import workloads as W
from test_gpu_mech import assert_state_equal, gpu_init, orc_init, params_pair

pytestmark = pytest.mark.gpu


def _engine(max_agents, max_ghosts=0):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    from paper_2503_10796_b200.bdm import TorchAllocator
    al = TorchAllocator(0)
    return Engine(0, max_agents, max_ghosts=max_ghosts, allocator=al), al


def test_create_ex_trajectory_bit_exact_and_blocks_returned(orc):
    cfg = W.CFG1
    eng, al = _engine(cfg.n)
    assert al.n_alloc >= 11 and al.n_free == 0          # the per-agent workspace (60 B/agent)
    assert al.bytes_live >= 60 * cfg.n
    a = gpu_init(eng, cfg)
    o = orc_init(orc, cfg)
    gp, op = params_pair(orc, cfg)
    for t in range(4):
        eng.step(a, gp, sync=True)
        st = eng.stats()
        o, cnt = orc.step_full(o, op)
        assert_state_equal(a.numpy(), o, f"create_ex step {t}")
        for k in ("cand", "nbr", "cont", "n_static"):
            assert st[k] == cnt[k], (t, k)
    n_before = al.n_alloc
    assert n_before > 11                                  # box starts, scan sums came from it too
    eng.close()
    assert al.n_free == al.n_alloc and al.bytes_live == 0 and not al.live


def test_create_ex_growth_goes_through_the_allocator(orc):
    """A context created too small regrows in bdm_grid_build: old blocks go back, new
    ones come from the callbacks, and the step is still the oracle's."""
    cfg = W.CFG2
    n = 30_011
    eng, al = _engine(1024)
    first = al.n_alloc
    a = gpu_init(eng, cfg, n)
    o = orc_init(orc, cfg, n)
    gp, op = params_pair(orc, cfg)
    for t in range(2):
        eng.step(a, gp, sync=True)
        o, _ = orc.step_full(o, op)
        assert_state_equal(a.numpy(), o, f"growth step {t}")
    assert al.n_alloc > first and al.n_free >= 11         # the 1,024-agent buffers were returned
    assert al.bytes_live >= 60 * n
    eng.close()
    assert al.bytes_live == 0 and not al.live


def test_create_ex_max_ghosts_sizes_the_sorted_workspace():
    """max_agents + max_ghosts entries per sorted array: a build of locals + ghosts of
    exactly that size re-allocates nothing per agent."""
    from paper_2503_10796_b200 import Agents
    cfg = W.CFG1
    eng, al = _engine(3000, max_ghosts=1096)
    assert al.bytes_live >= 60 * 4096
    a = gpu_init(eng, cfg, 4096)
    s = a.numpy()
    loc = Agents.from_numpy({k: v[:3000] for k, v in s.items()})
    gh = Agents.from_numpy({k: v[3000:] for k, v in s.items()})
    freed = al.n_free
    eng.grid_build(loc, 10.0, ghosts=gh)
    eng.sync()
    assert al.n_free - freed <= 2     # no regrowth of the 11 per-agent buffers (scan sums may)
    eng.close()
    assert not al.live


def test_create_ex_argument_checks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200.bdm import ALLOC_FN, FREE_FN, TorchAllocator, load_library
    lib = load_library()
    h = ctypes.c_void_p()
    al = TorchAllocator(0)
    assert lib.bdm_create_ex(ctypes.byref(h), 0, 10, -1, ALLOC_FN(0), FREE_FN(0), None) == -1
    assert lib.bdm_create_ex(ctypes.byref(h), 0, 10, 0, al.alloc_cb, FREE_FN(0), None) == -1
    failing = ALLOC_FN(lambda nbytes, st, user: None)
    freed = []
    rel = FREE_FN(lambda p, st, user: freed.append(p))
    assert lib.bdm_create_ex(ctypes.byref(h), 0, 10, 0, failing, rel, None) == -2  # BDM_ECAPACITY
    assert not h.value and not freed
