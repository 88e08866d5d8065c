"""Pins of the oracle's toroidal mechanics (boundary 2, reading R52): the
periodic cube [0, side)^3 of the paper's toroidal boundary ("agents that leave
the space on one side, will enter on the opposite side"), neighbours by minimum image
on the lattice of R19, positions wrapped by Alg. 9's literal rule (R20).

Pinned by: a pair across a face against the closed form of Eq. 4.1/4.2 at the pair's
periodic distance; wrap-around of a displaced agent; an all-pairs minimum-image brute
force in pure Python (forces to rounding, contact counts exactly); translation
invariance modulo the side; and the reduction to the open boundary for a cluster far
from every face."""
import math

import numpy as np
import pytest


def state(xs, ys, zs, ds):
    n = len(xs)
    return {"x": np.asarray(xs, np.float64), "y": np.asarray(ys, np.float64),
            "z": np.asarray(zs, np.float64), "d": np.asarray(ds, np.float64),
            "id": np.arange(n, dtype=np.uint32), "flags": np.full(n, 4, np.uint32)}


def torus(orc, side, **kw):
    return orc.mech_params(boundary=2, lo=(0.0, 0.0, 0.0), hi=(side, side, side), **kw)


def test_pair_across_a_face_closed_form(orc):
    """x = 1 and x = side - 1 are 2 apart through the face x = 0: Eq. 4.1/4.2 with
    delta = 10 - 2 = 8, rbar = 2.5: F_N = 2*8 - sqrt(20); the agent at x = 1 is pushed
    towards +x (away from its neighbour's image at -1), the other towards -x."""
    side = 100.0
    s = state([1.0, side - 1.0], [50.0, 50.0], [50.0, 50.0], [10.0, 10.0])
    out, cnt = orc.mech_step(s, torus(orc, side, dt=0.01, max_disp=3.0))
    Fn = 16.0 - math.sqrt(20.0)
    assert cnt["nbr"] == 2 and cnt["cont"] == 2
    assert abs(out["force"][0, 0] - Fn) <= 4 * math.ulp(Fn)
    assert out["force"][1, 0] == -out["force"][0, 0]
    assert out["force"][0, 1] == 0.0 and out["force"][0, 2] == 0.0
    assert abs(out["x"][0] - (1.0 + 0.01 * Fn)) <= 4 * math.ulp(1.2)
    assert abs(out["x"][1] - (side - 1.0 - 0.01 * Fn)) <= 4 * math.ulp(side)
    # the open boundary sees them 98 apart: no neighbours at all
    _, cnt_open = orc.mech_step(s, orc.mech_params(dt=0.01, max_disp=3.0))
    assert cnt_open["nbr"] == 0


def test_displaced_agent_wraps_around(orc):
    """An agent pushed across x = 0 re-enters at side - |x| (Alg. 9 wrap, exact here):
    agents at 0.5 and 2.5 overlap by 8, dt = 1 makes the displacement the 3 um cap."""
    side = 64.0
    s = state([0.5, 2.5], [32.0, 32.0], [32.0, 32.0], [10.0, 10.0])
    out, _ = orc.mech_step(s, torus(orc, side, dt=1.0, max_disp=3.0))
    assert out["x"][0] == side - 2.5      # 0.5 - 3 = -2.5 -> side - 2.5
    assert out["x"][1] == 5.5
    assert np.all((out["x"] >= 0.0) & (out["x"] < side))


def _brute_forces(s, side, k=2.0, gamma=1.0):
    """All pairs, minimum image per axis, Eq. 4.1/4.2 in plain Python floats."""
    n = len(s["x"])
    P = np.stack([s["x"], s["y"], s["z"]], 1)
    R = float(s["d"].max())
    F = np.zeros((n, 3))
    cont = 0
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            e = [float(P[i, a] - P[j, a]) for a in range(3)]
            e = [v - side if v > side / 2 else (v + side if v < -side / 2 else v) for v in e]
            D = e[0] * e[0] + e[1] * e[1] + e[2] * e[2]
            if D > R * R:
                continue
            dist = math.sqrt(D)
            ri, rj = s["d"][i] / 2, s["d"][j] / 2
            delta = (ri + rj) - dist
            if not (delta > 0 and dist > 0):
                continue
            cont += 1
            rbar = ri * rj / (ri + rj)
            fn = k * delta - gamma * math.sqrt(rbar * delta)
            for a in range(3):
                F[i, a] += fn / dist * e[a]
    return F, cont


@pytest.mark.parametrize("seed,n,side", [(1, 120, 40.0), (2, 300, 48.0), (3, 60, 36.1)])
def test_forces_equal_minimum_image_bruteforce(orc, seed, n, side):
    s = orc.init_spheres(n, seed, side, 8.0, 4.0, d_random=True)
    out, cnt = orc.mech_step(s, torus(orc, side))
    F, cont = _brute_forces(s, side)
    assert cnt["cont"] == cont
    scale = max(1.0, float(np.abs(F).max()))
    assert np.abs(out["force"] - F).max() <= 1e-12 * scale


def test_translation_invariance(orc):
    """Shifting every agent by t (mod side) shifts the result by t: the same contacts,
    forces to rounding (the summation order follows the shifted lattice)."""
    side = 50.0
    s = orc.init_spheres(400, 7, side, 8.0, 4.0, d_random=True)
    p = torus(orc, side)
    out, cnt = orc.mech_step(s, p)
    t = np.array([17.25, -3.5, 33.0])
    s2 = dict(s)
    for a, k in enumerate(("x", "y", "z")):
        s2[k] = np.array([orc.wrap(v + t[a], side) for v in s[k]])
    out2, cnt2 = orc.mech_step(s2, p)
    assert (cnt2["nbr"], cnt2["cont"]) == (cnt["nbr"], cnt["cont"])
    assert np.abs(out2["force"] - out["force"]).max() <= 1e-9 * max(1.0, np.abs(out["force"]).max())


def test_interior_cluster_matches_open_boundary(orc):
    """A cluster more than R from every face: no pair wraps, so the torus gives the
    open boundary's neighbours and forces (to the summation order of its own lattice)."""
    side = 400.0
    s = orc.init_spheres(500, 9, 60.0, 8.0, 4.0, d_random=True)
    for k in ("x", "y", "z"):
        s[k] = s[k] + 170.0
    out_t, cnt_t = orc.mech_step(s, torus(orc, side))
    out_o, cnt_o = orc.mech_step(s, orc.mech_params())
    assert (cnt_t["nbr"], cnt_t["cont"]) == (cnt_o["nbr"], cnt_o["cont"])
    assert np.abs(out_t["force"] - out_o["force"]).max() <= 1e-12 * max(1.0, np.abs(out_o["force"]).max())
    for k in ("x", "y", "z"):
        assert np.abs(out_t[k] - out_o[k]).max() <= 1e-12 * side


def test_invalid_torus_rejected(orc):
    s = state([1.0, 2.0], [1.0, 1.0], [1.0, 1.0], [10.0, 10.0])
    with pytest.raises(ValueError):
        orc.mech_step(s, torus(orc, 25.0))        # 2 boxes of edge >= 10 per axis
    with pytest.raises(ValueError):
        orc.mech_step(s, orc.mech_params(boundary=2, hi=(100.0, 100.0, 90.0)))  # not a cube
