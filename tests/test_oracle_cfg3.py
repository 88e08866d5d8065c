"""Pins for the oracle's growth + division pass (cfg3).

Alg. 4 control flow (algo:tumor_growth_module): grow while the diameter is
below the maximum, else divide; Cell::Divide splits the volume by the
volume ratio (0.5) and places the daughter along the division axis.  Checked against
exact cube roots (50-digit decimal), volume conservation, touching daughters, an
isotropy statistic of the axis and the population schedule derived independently
from the control flow.
"""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

getcontext().prec = 50
V_MAX = (math.pi / 6.0) * 1728.0


def dcbrt(v: float) -> Decimal:
    x = Decimal(v)
    y = Decimal(v) ** (Decimal(1) / Decimal(3))
    for _ in range(5):  # polish
        y = (2 * y + x / (y * y)) / 3
    return y


def test_cbrt_det_exact_cubes(orc):
    for v, r in ((8.0, 2.0), (27.0, 3.0), (0.125, 0.5), (1000.0, 10.0), (64.0, 4.0),
                 (2.0**60, 2.0**20), (2.0**-30, 2.0**-10)):
        assert orc.cbrt_det(v) == r, v


def test_cbrt_det_within_two_ulp(orc):
    rng = np.random.default_rng(1)
    for v in np.exp(rng.uniform(-40, 40, 3000)):
        got = orc.cbrt_det(float(v))
        want = dcbrt(float(v))
        assert float(abs(Decimal(got) - want)) <= 2 * math.ulp(float(want)), v  # R28: ulp level


def test_division_axis_unit_and_isotropic(orc):
    U = np.array([orc.division_axis(1, i, 7) for i in range(20000)])
    nrm = np.linalg.norm(U, axis=1)
    assert np.all(np.abs(nrm - 1.0) <= 4e-16)
    assert np.all(np.abs(U.mean(0)) < 5 * math.sqrt(1 / 3 / 20000))
    assert np.all(np.abs((U**2).mean(0) - 1 / 3) < 0.02)
    # deterministic per (seed, id, step), different for another step
    assert np.array_equal(orc.division_axis(1, 5, 3), orc.division_axis(1, 5, 3))
    assert not np.array_equal(orc.division_axis(1, 5, 3), orc.division_axis(1, 5, 4))


def _state(orc, n, seed=1, side=1000.0):
    s = orc.init_spheres(n, seed, side, 8.0)
    s["vol"] = orc.init_volumes(s)
    return s


def test_growth_diameter_closed_form(orc):
    """First growth of a d = 8 sphere: d' = 2 cbrt((pi/6 * 512 + 400) * 0.75/pi)."""
    s = _state(orc, 1)
    out = orc.grow_divide(s, 400.0, V_MAX, 1, 0)
    want = 2 * dcbrt(((math.pi / 6.0) * 512.0 + 400.0) * (0.75 / math.pi))
    assert float(abs(Decimal(out["d"][0]) - want)) <= 2 * math.ulp(10.8)
    assert out["flags"][0] & orc.GREW
    assert abs(out["d"][0] - 10.846189143068989) < 1e-12   # SURVEY 9.2 table, step 2 d


def test_division_conserves_volume_and_touches(orc):
    s = _state(orc, 50)
    s["vol"][:] = 1100.0           # everyone divides
    s["flags"][:] = 0
    out = orc.grow_divide(s, 400.0, V_MAX, 1, 9)
    assert len(out["x"]) == 100
    assert np.array_equal(out["id"], np.arange(100, dtype=np.uint32))
    for i in range(50):
        j = 50 + i
        assert out["vol"][i] + out["vol"][j] == 1100.0      # V/2 + V/2 = V exactly
        dist = math.dist((out["x"][i], out["y"][i], out["z"][i]),
                         (out["x"][j], out["y"][j], out["z"][j]))
        r = out["d"][i] / 2
        assert abs(dist - 2 * r) <= 1e-12 * r                # daughters just touch
        want_r = dcbrt(550.0 * (0.75 / math.pi))
        assert float(abs(Decimal(r) - want_r)) <= 2 * math.ulp(r)
        # mother and daughter straddle the pre-division centre along the axis
        u = orc.division_axis(1, i, 9)
        mid = np.array([out["x"][i] + out["x"][j], out["y"][i] + out["y"][j],
                        out["z"][i] + out["z"][j]]) / 2
        assert np.allclose(mid, [s["x"][i], s["y"][i], s["z"][i]], atol=1e-12)
        assert np.allclose(np.array([out["x"][j] - out["x"][i], out["y"][j] - out["y"][i],
                                     out["z"][j] - out["z"][i]]) / (2 * r), u, atol=1e-12)
    assert np.all(out["flags"][:50] & orc.MOVED)
    assert np.all(out["flags"][50:] == orc.ADDED)


def _schedule_from_control_flow(steps):
    """Population after each step for equal spheres starting at d = 8: Alg. 4's
    'grow while d < 12, else divide' evaluated on exact cube roots (decimal)."""
    V = Decimal(math.pi) / 6 * 512
    Vmax = Decimal(math.pi) / 6 * 1728
    n, out = 1, []
    for _ in range(steps):
        d = 2 * (V * Decimal(0.75) / Decimal(math.pi)) ** (Decimal(1) / Decimal(3))
        if d < 12 and V < Vmax:
            V += 400
        else:
            V /= 2
            n *= 2
        out.append(n)
    return out


def test_population_schedule(orc):
    """1,1,2,2,4,4,4,8,8,16,16,32,... independent of the mechanics."""
    steps = 12
    want = _schedule_from_control_flow(steps)
    assert want[:12] == [1, 1, 2, 2, 4, 4, 4, 8, 8, 16, 16, 32]
    s = _state(orc, 300, side=300.0)
    p = orc.mech_params()
    for t in range(steps):
        s, _ = orc.cfg3_step(s, p, 400.0, V_MAX, 1, t)
        assert len(s["x"]) == 300 * want[t], t
        assert np.array_equal(np.sort(s["id"]), np.arange(len(s["x"]), dtype=np.uint32))
        # all diameters are equal at each step (synchronised cycle)
        assert np.ptp(s["d"]) == 0.0
