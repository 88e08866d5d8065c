"""GPU parity for row f3 (delta-encoded + LZ4 aura messages) through the C
ABI against the pinned oracle (tests/test_oracle_aura.py): the reference order, the
stream bytes (the greedy parse is deterministic, so the streams are identical), decoding
of the oracle's streams, round trips, malformed streams and capacity errors."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

FIELDS = ("x", "y", "z", "d", "id", "flags")


@pytest.fixture(scope="module")
def eng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    e = Engine(0, 1 << 12)
    yield e
    e.close()


def _dev(s, capacity=None):
    from paper_2503_10796_b200 import Agents
    n = len(s["x"])
    if n == 0:
        a = Agents.empty(max(capacity or 1, 1))
        a.n = 0
        return a
    return Agents.from_numpy({k: np.asarray(s[k]) for k in FIELDS}, capacity=capacity)


def _host(a):
    g = a.numpy()
    return {k: g[k] for k in FIELDS}


def _same(a, b, what=""):
    for k in FIELDS:
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), (what, k)


def _slab_aura(orc, n, steps, margin=12.0, seed=0):
    """Agents of a cfg2-like cube within `margin` of the plane x = side/2, before and
    after `steps` mechanics steps (the aura a slab neighbour receives)."""
    cfg = W.cfg2_scaled(n)
    s = orc.init_spheres(cfg.n, cfg.seed + seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    op = orc.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                         force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    mid = 0.5 * cfg.side
    out = []
    for t in range(steps + 1):
        sel = np.abs(s["x"] - mid) < margin
        out.append({k: np.ascontiguousarray(np.asarray(s[k])[sel]) for k in FIELDS})
        if t < steps:
            s, _ = orc.step_full(s, op)
    return out[0], out[-1]


def _encode(eng, msg, ref):
    import torch
    m, r = _dev(msg), _dev(ref)
    cap = eng.aura_max_size(len(ref["x"]), len(msg["x"]))
    buf = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    k = eng.aura_encode(m, r, buf)
    return buf[:k].cpu().numpy().tobytes()


def _liblz4_pin(orc, st, msg, ref):
    """The GPU stream decodes under the LZ4 reference decoder (liblz4) to exactly the
    oracle's payload: losslessness pinned independently of the parse convention (R50)."""
    import lz4_ref
    if lz4_ref.lib() is None:
        pytest.skip("liblz4 not installed")
    pay, nnew = orc.aura_payload(msg, ref)
    got, nref, nnew2 = lz4_ref.decode_stream(st)
    assert got == bytes(pay)
    assert (nref, nnew2) == (len(ref["id"]), nnew)


def test_reference_is_id_order(eng, orc):
    rng = np.random.default_rng(1)
    n = 5000
    msg = {"x": rng.uniform(0, 9, n), "y": rng.uniform(0, 9, n), "z": rng.uniform(0, 9, n),
           "d": rng.uniform(8, 12, n), "id": rng.permutation(4 * n)[:n].astype(np.uint32),
           "flags": rng.integers(0, 99, n).astype(np.uint32)}
    from paper_2503_10796_b200 import Agents
    r = Agents.empty(n)
    eng.aura_reference(_dev(msg), r)
    _same(_host(r), orc.aura_reference(msg))


@pytest.mark.parametrize("n", [0, 1, 31, 2048, 2049, 70_001, 1_000_003])
def test_reference_radix_sort_full_id_range(eng, n):
    """The hand-written LSD radix sort behind bdm_aura_reference: unique ids drawn over
    the whole 32-bit range (every digit of every pass is exercised), sizes around the
    2,048-pair tile and many tiles with a ragged tail; every field follows its id.
    Expected values from numpy's argsort (ids are unique, so the order is unique)."""
    from paper_2503_10796_b200 import Agents
    rng = np.random.default_rng(100 + n)
    pool = np.unique(rng.integers(0, 2 ** 32, int(1.1 * n) + 8, dtype=np.uint64).astype(np.uint32))
    pool = pool[(pool != 0) & (pool != 0xFFFFFFFF)]
    ids = rng.permutation(pool)[:n]
    if n > 2:
        ids[0], ids[1] = np.uint32(0xFFFFFFFF), np.uint32(0)   # both ends of the key range
    ids = rng.permutation(ids)
    assert len(ids) == n
    msg = {"x": rng.uniform(0, 9, n), "y": rng.uniform(0, 9, n), "z": rng.uniform(0, 9, n),
           "d": rng.uniform(8, 12, n), "id": ids, "flags": rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)}
    r = Agents.empty(max(n, 1))
    eng.aura_reference(_dev(msg, capacity=max(n, 1)), r)
    got = _host(r)
    order = np.argsort(ids, kind="stable")
    assert r.n == n
    for k in FIELDS:
        assert np.array_equal(np.asarray(got[k])[:n].view(np.uint8), np.ascontiguousarray(msg[k][order]).view(np.uint8)), k


@pytest.mark.parametrize("case", ["moved", "identical", "no_reference", "empty_message", "churn"])
def test_stream_bytes_equal_oracle_and_round_trip(eng, orc, case):
    before, after = _slab_aura(orc, 30000, 2)
    ref = orc.aura_reference(before)
    msg = after
    if case == "identical":
        msg = before
    elif case == "no_reference":
        ref = {k: v[:0] for k, v in ref.items()}
    elif case == "empty_message":
        msg = {k: v[:0] for k, v in msg.items()}
    elif case == "churn":  # a third left the aura, new agents joined
        rng = np.random.default_rng(5)
        keep = rng.random(len(msg["x"])) < 0.67
        extra = {k: np.asarray(v)[:400].copy() for k, v in before.items()}
        extra["id"] = extra["id"] + np.uint32(10_000_000)
        msg = {k: np.concatenate([np.asarray(msg[k])[keep], extra[k]]) for k in FIELDS}
    st_o = orc.aura_encode(msg, ref)
    st_g = _encode(eng, msg, ref)
    _liblz4_pin(orc, st_g, msg, ref)                      # the reference decoder's pin
    assert st_g == st_o                                   # identical streams (convention)
    import torch
    from paper_2503_10796_b200 import Agents
    r = _dev(ref)
    out = Agents.empty(max(len(msg["x"]), 1))
    buf = torch.frombuffer(bytearray(st_o), dtype=torch.uint8).cuda()
    eng.aura_decode(buf, len(st_o), r, out)
    _same(_host(out), orc.aura_decode(st_o, ref), case)   # decode = oracle decode
    got = _host(out)
    assert sorted(got["id"].tolist()) == sorted(np.asarray(msg["id"]).tolist())


def test_multi_chunk_ragged_and_ratio(eng, orc):
    """~100k-agent payload (> 900 chunks with a ragged last chunk): identical streams; the
    delta stream of a real slab aura is much smaller than the raw 40 B/agent and than
    LZ4 alone (the paper: 3.0-5.2x from LZ4, another 1.1-3.5x from the delta)."""
    before, after = _slab_aura(orc, 400_000, 1, margin=12.0, seed=3)
    ref = orc.aura_reference(before)
    st_o = orc.aura_encode(after, ref)
    st_g = _encode(eng, after, ref)
    _liblz4_pin(orc, st_g, after, ref)
    assert st_g == st_o
    plain = _encode(eng, after, {k: v[:0] for k, v in ref.items()})
    raw = 40 * len(after["x"])
    assert len(st_g) < len(plain) < raw


def test_malformed_and_capacity_errors(eng, orc):
    import torch
    from paper_2503_10796_b200 import Agents, BdmError
    before, after = _slab_aura(orc, 20000, 1)
    ref = orc.aura_reference(before)
    st = orc.aura_encode(after, ref)
    r = _dev(ref)
    out = Agents.empty(len(after["x"]) + 8)
    buf = torch.frombuffer(bytearray(st), dtype=torch.uint8).cuda()
    with pytest.raises(BdmError):                       # truncated
        eng.aura_decode(buf, len(st) - 7, r, out)
    bad = bytearray(st)
    bad[40:44] = (0xFFFFFF).to_bytes(4, "little")       # chunk 0 claims 16 MB
    with pytest.raises(BdmError):
        eng.aura_decode(torch.frombuffer(bad, dtype=torch.uint8).cuda(), len(bad), r, out)
    bad = bytearray(st)
    bad[0] ^= 1                                         # magic
    with pytest.raises(BdmError):
        eng.aura_decode(torch.frombuffer(bad, dtype=torch.uint8).cuda(), len(bad), r, out)
    bad = bytearray(st)
    k0 = int.from_bytes(st[40:44], "little")
    nch = int.from_bytes(st[32:36], "little")
    bad[40 + 4 * nch] = 0xF0                             # chunk 0: a literal run past its end
    bad[40 + 4 * nch + 1] = 0xFF
    assert k0 > 2
    with pytest.raises(BdmError):
        eng.aura_decode(torch.frombuffer(bad, dtype=torch.uint8).cuda(), len(bad), r, out)
    r_other = _dev({k: v[:-1] for k, v in ref.items()})
    with pytest.raises(BdmError):                       # another reference
        eng.aura_decode(buf, len(st), r_other, out)
    small = Agents.empty(4)
    with pytest.raises(BdmError):
        eng.aura_decode(buf, len(st), r, small)
    tiny = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(BdmError):                       # stream buffer too small
        eng.aura_encode(_dev(after), r, tiny)
    eng.aura_decode(buf, len(st), r, out)               # the context still works
    _same(_host(out), orc.aura_decode(st, ref))
