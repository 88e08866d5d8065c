"""Pins for the CPU oracle (runs without a GPU).

Every test here checks oracle/ against something other than itself: a library routine
(ATen's Philox engine), closed forms of Eq. 4.1 evaluated in 50-digit decimal
arithmetic (tests/golden/eq41_closed_forms.json), the paper's Morton worked example
(tests/golden/morton_2d_3x3.txt), brute force on tiny inputs (pure Python), and
invariants (antisymmetry, net force, cap, static transparency, sortedness).
"""
import itertools
import json
import math
import os
import shutil
import subprocess
import tempfile
from decimal import Decimal, getcontext

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
getcontext().prec = 50


def ulps(a: float, b: Decimal) -> float:
    """|a - b| in units of the last place of b (as a float)."""
    bf = float(b)
    if bf == 0.0:
        return abs(a) / 5e-324
    return float(abs(Decimal(a) - b)) / math.ulp(bf)


def state(xs, ys=None, zs=None, ds=None, flags=None):
    n = len(xs)
    s = {
        "x": np.asarray(xs, np.float64),
        "y": np.asarray(ys if ys is not None else [0.0] * n, np.float64),
        "z": np.asarray(zs if zs is not None else [0.0] * n, np.float64),
        "d": np.asarray(ds if ds is not None else [10.0] * n, np.float64),
        "id": np.arange(n, dtype=np.uint32),
        "flags": np.asarray(flags if flags is not None else [4] * n, np.uint32),
    }
    return s


# ------------------------------------------------------------------ Philox (R22)
ATEN_PROG = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  for (int a = 1; a + 2 < argc; a += 3) {
    at::philox_engine e(strtoull(argv[a], 0, 0), strtoull(argv[a + 1], 0, 0),
                        strtoull(argv[a + 2], 0, 0));
    for (int i = 0; i < 4; i++) printf("%u\n", e());
  }
}
"""


def _aten_philox_binary():
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    d = tempfile.mkdtemp(prefix="bdm_philox_")
    src = os.path.join(d, "p.cpp")
    with open(src, "w") as f:
        f.write(ATEN_PROG)
    exe = os.path.join(d, "p")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", inc, src, "-o", exe])
    return d, exe


def test_philox_matches_aten_engine(orc):
    """Oracle Philox4x32-10 == ATen's header-only philox_engine (a library routine).

    ATen's counter is (offset_lo, offset_hi, subsequence_lo, subsequence_hi) and its
    key is the 64-bit seed, so our counter (c0, c1, c2, c3) maps to
    offset = c0 | c1 << 32, subsequence = c2 | c3 << 32."""
    if shutil.which("g++") is None:
        pytest.skip("g++ missing")
    d, exe = _aten_philox_binary()
    try:
        rng = np.random.default_rng(7)
        cases = [((0, 0, 0, 0), 0), ((0xFFFFFFFF,) * 4, 0xFFFFFFFFFFFFFFFF),
                 ((5, 0, 0xFFFFFFFF, 2), 1), ((123, 0, 17, 3), 1)]
        for _ in range(40):
            c = tuple(int(v) for v in rng.integers(0, 2**32, 4, dtype=np.uint64))
            cases.append((c, int(rng.integers(0, 2**63))))
        args = []
        for c, seed in cases:
            args += [str(seed), str(c[2] | (c[3] << 32)), str(c[0] | (c[1] << 32))]
        out = subprocess.check_output([exe, *args]).decode().split()
        ref = np.array([int(v) for v in out], dtype=np.uint64).reshape(-1, 4)
        for (c, seed), r in zip(cases, ref):
            got = orc.philox4x32_10(c, (seed & 0xFFFFFFFF, seed >> 32))
            assert list(got) == list(r), (c, seed)
    finally:
        shutil.rmtree(d, ignore_errors=True)


def test_u53_u32_exact(orc):
    """R29: u53 = ((wa>>5)*2^26 + (wb>>6)) * 2^-53 and u32 = w*2^-32, both exact."""
    assert orc.u53(0, 0) == 0.0
    assert orc.u53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0**-53
    assert orc.u53(1 << 5, 0) == 2.0**-27
    assert orc.u53(0, 1 << 6) == 2.0**-53
    assert orc.u32(0) == 0.0 and orc.u32(0xFFFFFFFF) == 1.0 - 2.0**-32
    assert orc.u32(1 << 31) == 0.5


def test_init_uniform_moments(orc):
    """Uniform-in-cube init: first two moments within 5 sigma, ids dense,
    flags = ADDED, diameters in [8, 12)."""
    n, side = 200_000, 100.0
    s = orc.init_spheres(n, 1, side, 8.0, 4.0, d_random=True)
    for a in ("x", "y", "z"):
        v = s[a]
        assert v.min() >= 0.0 and v.max() < side
        sig = side / math.sqrt(12.0) / math.sqrt(n)
        assert abs(v.mean() - side / 2) < 5 * sig
        assert abs(v.var() - side**2 / 12) < 5 * side**2 / 12 * math.sqrt(0.8 / n)
    assert s["d"].min() >= 8.0 and s["d"].max() < 12.0
    assert abs(s["d"].mean() - 10.0) < 5 * (4 / math.sqrt(12) / math.sqrt(n))
    assert np.array_equal(s["id"], np.arange(n, dtype=np.uint32))
    assert np.all(s["flags"] == orc.ADDED)
    # per-id generation: a shifted id range reproduces the same agents
    t = orc.init_spheres(100, 1, side, 8.0, 4.0, d_random=True, id0=500)
    for a in ("x", "y", "z", "d"):
        assert np.array_equal(t[a], s[a][500:600])
    # independence of the three coordinate streams (correlation ~ 0)
    assert abs(np.corrcoef(s["x"], s["y"])[0, 1]) < 0.02
    assert abs(np.corrcoef(s["x"], s["z"])[0, 1]) < 0.02


# ------------------------------------------------------------------ Morton (A12)
def test_morton_paper_worked_example(orc):
    with open(os.path.join(GOLDEN, "morton_2d_3x3.txt")) as f:
        want = [int(v) for line in f if not line.startswith("#") for v in line.split()]
    got = sorted(orc.morton([x, y], 2) for x in range(3) for y in range(3))
    assert got == want


def test_morton_3d_bit_order(orc):
    """x in the lowest bit: m(1,0,0)=1, m(0,1,0)=2, m(0,0,1)=4, m(1,1,1)=7, m(2,0,0)=8."""
    assert orc.morton([1, 0, 0], 2) == 1
    assert orc.morton([0, 1, 0], 2) == 2
    assert orc.morton([0, 0, 1], 2) == 4
    assert orc.morton([1, 1, 1], 2) == 7
    assert orc.morton([2, 0, 0], 2) == 8
    assert orc.morton([3, 3, 3], 2) == 63
    # 2D: (1,1) -> 3 (SPEC example S:~250), (2,0) -> 4
    assert orc.morton([1, 1], 2) == 3 and orc.morton([2, 0], 2) == 4


def test_blocked_key_bijective_and_tile_contiguous(orc):
    D = (9, 6, 5)
    T = [(v + 3) // 4 for v in D]
    keys = {}
    for bx, by, bz in itertools.product(range(D[0]), range(D[1]), range(D[2])):
        k = orc.blocked_key(bx, by, bz, D)
        assert k not in keys
        keys[k] = (bx, by, bz)
        assert k < T[0] * T[1] * T[2] * 64
        # tile = k // 64 is the row-major tile index; k % 64 the in-tile Morton code
        tile = ((bz // 4) * T[1] + by // 4) * T[0] + bx // 4
        assert k // 64 == tile
        assert k % 64 == orc.morton([bx % 4, by % 4, bz % 4], 2)


# ------------------------------------------------------------------ Eq. 4.1 closed forms
def _golden():
    with open(os.path.join(GOLDEN, "eq41_closed_forms.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: c["name"])
def test_eq41_closed_forms(orc, case):
    c1 = [float(Decimal(v)) for v in case["c1"]]
    c2 = [float(Decimal(v)) for v in case["c2"]]
    s = state([c1[0], c2[0]], [c1[1], c2[1]], [c1[2], c2[2]],
              [2.0 * case["r1"], 2.0 * case["r2"]])
    p = orc.mech_params(dt=0.01, max_disp=3.0)
    out, cnt = orc.mech_step(s, p)
    F = out["force"]
    Fn = Decimal(case["F_N"])
    want = [Decimal(v) for v in case["force_on_1"]]
    for a in range(3):
        if want[a] == 0:
            assert F[0, a] == 0.0
        else:
            assert ulps(F[0, a], want[a]) <= 4, (a, F[0, a], want[a])
        # antisymmetry f_21 = -f_12, bitwise (same D, same F_N, negated d*)
        assert F[1, a] == -F[0, a]
    assert cnt["nbr"] == 2
    if Fn == 0:
        # exact zero: contact but no force, no motion, nnz stays 0
        assert cnt["cont"] == 2
        assert np.all(F == 0.0)
        assert out["x"][0] == s["x"][0] and out["flags"][0] == 0
    else:
        assert (int(out["flags"][0]) >> orc.NNZ_SHIFT) & 3 == 1
        assert out["flags"][0] & orc.MOVED
    if case["name"] == "max_attraction":
        assert F[0, 0] > 0 and out["x"][0] > 0.0          # pulled towards +x
        assert abs(out["x"][0] - 0.003125) <= 2 * math.ulp(0.003125)
    if case["name"] == "equal_radii_delta1":
        d0 = out["x"][0] - s["x"][0]
        d1 = out["x"][1] - s["x"][1]
        assert ulps(-d0, Decimal("0.01") * Fn) <= 8          # 0.004188611699158103...
        assert abs(d0 + d1) <= 2 * math.ulp(9.0)             # equal and opposite
    if case["name"] == "cap_case":
        # uncapped |dt F| = 5.98 > 3: displacement capped to exactly max_disp (<= 1 ulp)
        d0 = out["x"][0] - s["x"][0]
        assert abs(d0 + 3.0) <= math.ulp(3.0)
        assert out["y"][0] == 0.0 and out["z"][0] == 0.0


def test_superposition_collinear(orc):
    g = _golden()["collinear_middle"]
    xs = [float(Decimal(v)) for v in g["x"]]
    s = state(xs)
    out, _ = orc.mech_step(s, orc.mech_params())
    assert ulps(out["force"][1, 0], Decimal(g["sum"])) <= 8
    # symmetric configuration: the two terms cancel up to the accumulation rounding,
    # nnz = 2 so condition (iv) keeps the middle agent non-static forever
    s = state([0.0, 9.0, 18.0])
    p = orc.mech_params(detect_static=True, force_threshold=1e-6)
    for step in range(4):
        out, cnt = orc.mech_step(s, p)
        Fm = out["force"][1, 0]
        # step 0 is exactly symmetric; later steps carry the rounding of x +/- Delta
        tol = 2 * math.ulp(0.42) if step == 0 else 1e-12
        assert abs(Fm) <= tol
        assert (int(out["flags"][1]) >> orc.NNZ_SHIFT) & 3 == 2
        assert not (out["flags"][1] & orc.STATIC)
        s = dict(s, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])


# ------------------------------------------------------------------ neighbour sets
def _random_state(orc, n, seed, side, dlo=8.0, dw=4.0):
    return orc.init_spheres(n, seed, side, dlo, dw, d_random=True)


def test_neighbors_grid_equals_bruteforce_200_seeds(orc):
    """The grid's 27-box enumeration reaches exactly the all-pairs relation
    (P:4506-4511 vs the plain definition)."""
    rng = np.random.default_rng(3)
    for seed in range(200):
        n = int(rng.integers(0, 1000))
        side = float(rng.uniform(10.0, 150.0))
        s = _random_state(orc, n, seed + 1, side)
        R = float(s["d"].max()) if n else 0.0
        a = orc.neighbor_pairs_grid(s)
        b = orc.neighbor_pairs_brute(s, R)
        assert np.array_equal(a, b), seed


def test_neighbors_pure_python_bruteforce(orc):
    """Independent pure-Python all-pairs recount on tiny inputs."""
    for seed in (1, 2, 3, 17):
        s = _random_state(orc, 90, seed, 40.0)
        R = float(s["d"].max())
        want = set()
        X, Y, Z = s["x"].tolist(), s["y"].tolist(), s["z"].tolist()
        for i in range(90):
            for j in range(90):
                if i != j:
                    dd = (X[i] - X[j]) ** 2 + (Y[i] - Y[j]) ** 2 + (Z[i] - Z[j]) ** 2
                    if dd <= R * R:
                        want.add((i << 32) | j)
        got = set(int(v) for v in orc.neighbor_pairs_grid(s))
        assert got == want
        # symmetric relation
        assert all(((p & 0xFFFFFFFF) << 32 | (p >> 32)) in got for p in got)


def test_grid_geometry_covers_agents(orc):
    s = _random_state(orc, 3000, 5, 120.0)
    R, L, o, D = orc.grid_geometry(s)
    assert R == s["d"].max() and L == R * (1 + 2.0**-20) and L > R
    assert np.array_equal(o, [s["x"].min(), s["y"].min(), s["z"].min()])
    for a, key in enumerate(("x", "y", "z")):
        b = np.floor((s[key] - o[a]) / L)
        assert b.min() == 0 and b.max() == D[a] - 1


# ------------------------------------------------------------------ invariants of the step
def test_net_internal_force_vanishes(orc):
    """Antisymmetry f_ij = -f_ji => sum_i F_i = 0 up to accumulation rounding:
    |sum F| <= (max_i n_i + 1) * 2^-53 * sum_ij |f_ij| (Neumaier outer sum)."""
    s = _random_state(orc, 3000, 11, 110.0)
    p = orc.mech_params(dt=1.0, max_disp=1e300)
    out, cnt = orc.mech_step(s, p)
    F = out["force"]
    pairs = orc.neighbor_pairs_brute(s, float(s["d"].max()))
    i = (pairs >> np.uint64(32)).astype(np.int64)
    j = (pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)
    tot = 0.0
    for a, b in zip(i.tolist(), j.tolist()):
        D = (s["x"][a] - s["x"][b]) ** 2 + (s["y"][a] - s["y"][b]) ** 2 + (s["z"][a] - s["z"][b]) ** 2
        Fn, sc, contact = orc.pair_force(2.0, 1.0, D, s["d"][a] / 2, s["d"][b] / 2)
        tot += abs(Fn)
    nmax = np.bincount(i).max()
    bound = (nmax + 1) * 2.0**-53 * tot
    for a in range(3):
        total = math.fsum(F[:, a].tolist())
        assert abs(total) <= bound, (a, total, bound)
    assert cnt["cont"] > 1000


def test_two_agent_antisymmetry_random(orc):
    rng = np.random.default_rng(5)
    for _ in range(200):
        c = rng.uniform(0, 10, (2, 3))
        s = state(c[:, 0], c[:, 1], c[:, 2], rng.uniform(4, 12, 2))
        out, _ = orc.mech_step(s, orc.mech_params(max_disp=1e300))
        assert np.array_equal(out["force"][0], -out["force"][1])


def test_displacement_cap_invariant(orc):
    """|Delta| <= max_disp (+1 ulp), and capped displacements are parallel to F."""
    s = _random_state(orc, 2000, 9, 60.0)   # very dense: many capped agents
    p = orc.mech_params(dt=0.5, max_disp=3.0)
    out, _ = orc.mech_step(s, p)
    Dl = np.stack([out["x"] - s["x"], out["y"] - s["y"], out["z"] - s["z"]], 1)
    nrm = np.sqrt((Dl**2).sum(1))
    assert nrm.max() <= 3.0 * (1 + 1e-12)
    capped = np.linalg.norm(0.5 * out["force"], axis=1) > 3.0
    assert capped.sum() > 100
    cosang = (Dl[capped] * out["force"][capped]).sum(1) / (nrm[capped] * np.linalg.norm(out["force"][capped], axis=1))
    assert np.all(cosang > 1 - 1e-9)
    assert np.allclose(nrm[capped], 3.0, rtol=1e-12)


def test_isolated_agent_is_static_and_unchanged(orc):
    s = state([0.0], ds=[10.0])
    p = orc.mech_params(detect_static=True)
    out, cnt = orc.mech_step(s, p)      # step 0: ADDED, so not static
    assert cnt["n_static"] == 0 and out["x"][0] == 0.0 and out["flags"][0] == 0
    s = dict(s, flags=out["flags"])
    out, cnt = orc.mech_step(s, p)      # step 1: static
    assert cnt["n_static"] == 1 and out["flags"][0] == orc.STATIC
    assert out["x"][0] == 0.0 and np.all(out["force"] == 0)


def _run(orc, s, p, steps):
    traj = []
    stats = []
    for _ in range(steps):
        out, cnt = orc.mech_step(s, p)
        s = dict(s, x=out["x"], y=out["y"], z=out["z"], flags=out["flags"])
        traj.append((s["x"].copy(), s["y"].copy(), s["z"].copy()))
        stats.append(cnt)
    return traj, stats


@pytest.mark.parametrize("side,tau", [(160.0, 1e-3), (640.0, 0.0), (160.0, 0.05)])
def test_static_skip_is_transparent(orc, side, tau):
    """'safe to skip the expensive force calculation': trajectories with
    the static-agent skip on and off are bit-identical."""
    s = orc.init_spheres(4096, 1, side, 10.0)
    on, st_on = _run(orc, s, orc.mech_params(detect_static=True, force_threshold=tau), 10)
    off, st_off = _run(orc, s, orc.mech_params(detect_static=False, force_threshold=tau), 10)
    for a, b in zip(on, off):
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    assert sum(c["n_static"] for c in st_on) > 100     # the skip actually fired
    assert sum(c["cand"] for c in st_on) < sum(c["cand"] for c in st_off)


def test_sample_mode_equals_full_mode(orc):
    s = _random_state(orc, 5000, 2, 150.0)
    s["flags"][::3] = 0
    p = orc.mech_params(detect_static=True)
    full, _ = orc.mech_step(s, p)
    idx = np.random.default_rng(0).choice(5000, 700, replace=False)
    part, _ = orc.mech_step(s, p, sample=idx)
    for k in ("x", "y", "z", "flags", "force"):
        assert np.array_equal(part[k], full[k][idx])


def test_sorted_order_invariants(orc):
    s = _random_state(orc, 6000, 4, 170.0)
    perm, keys = orc.sorted_order(s)
    assert np.array_equal(np.sort(perm), np.arange(6000))
    assert np.all(np.diff(keys.astype(np.int64)) >= 0)
    ids = s["id"][perm]
    same = keys[1:] == keys[:-1]
    assert np.all(ids[1:][same] > ids[:-1][same])
    R, L, o, D = orc.grid_geometry(s)
    for t in range(0, 6000, 97):
        i = perm[t]
        b = [int(math.floor((s[a][i] - o[k]) / L)) for k, a in enumerate("xyz")]
        assert keys[t] == orc.blocked_key(*b, D)


def test_empty_and_single(orc):
    s = state([])
    out, cnt = orc.mech_step(s, orc.mech_params())
    assert len(out["x"]) == 0 and cnt["cand"] == 0
    assert len(orc.neighbor_pairs_grid(s)) == 0
