"""Pins of the oncology oracle (Alg. 4 algo:tumor_growth_module,
P:3067-3112, Table 4.2; agent removal P:4545-4603) against what the algorithm
fixes, without re-evaluating its formulas: unit-length Brownian steps and their isotropy,
exact age / volume bookkeeping, the age gate of apoptosis, death and division
frequencies within 5 sigma, volume conservation and touching daughters, removal keeping
the survivors' data and order, fresh unique ids, population accounting."""
import math

import numpy as np
import pytest

import oracle as orc


def _pop(n, seed=1, side=200.0, d=10.0, ages=None):
    s = orc.init_spheres(n, seed, side, d, 0.0, False)
    s["vol"] = (math.pi / 6.0) * s["d"] ** 3
    s["age"] = np.asarray(ages if ages is not None else np.zeros(n), np.uint32)
    return s


def test_brownian_steps_are_unit_and_isotropic():
    n = 20000
    s = _pop(n)
    p = orc.onco_params(displacement_rate=0.5, max_diameter=0.0, p_death=0.0, p_div=0.0, step=3)
    out, nxt = orc.onco_step(s, p, n)
    assert nxt == n and len(out["x"]) == n
    assert np.array_equal(out["id"], s["id"])            # order and ids kept
    dx = np.stack([out[c] - s[c] for c in ("x", "y", "z")])
    r = np.sqrt((dx ** 2).sum(axis=0))
    assert np.all(np.abs(r - 0.5) <= 1e-12)               # |brownian| = 1 (R41)
    sig = 0.5 / math.sqrt(3 * n)
    assert np.all(np.abs(dx.mean(axis=1)) < 5 * sig)      # isotropic: mean 0
    m2 = (dx ** 2).mean(axis=1)                           # E[dx^2] = rate^2 / 3
    assert np.all(np.abs(m2 - 0.25 / 3) < 5 * math.sqrt(0.25 ** 2 * (1 / 5 - 1 / 9) / n))
    assert np.array_equal(out["age"], s["age"] + 1)
    assert np.all(out["flags"] & orc.MOVED)


def test_age_gate_and_certain_death():
    n = 1000
    ages = np.where(np.arange(n) % 3 == 0, 87, 86)          # a third at the minimum age
    s = _pop(n, ages=ages)
    p = orc.onco_params(p_death=1.0, p_div=0.0, step=1)
    out, _ = orc.onco_step(s, p, n)
    keep = ages < 87
    assert len(out["x"]) == keep.sum()
    assert np.array_equal(out["id"], s["id"][keep])         # survivors keep their order
    assert np.array_equal(out["age"], ages[keep] + 1)


def test_death_frequency():
    n = 40000
    s = _pop(n, ages=np.full(n, 200))
    p = orc.onco_params(p_death=0.25, p_div=0.0, step=7)
    out, _ = orc.onco_step(s, p, n)
    dead = n - len(out["x"])
    assert abs(dead - 0.25 * n) < 5 * math.sqrt(n * 0.25 * 0.75)


def test_growth_bookkeeping():
    n = 500
    s = _pop(n)
    p = orc.onco_params(growth=42.0, max_diameter=14.0, p_death=0.0, step=2)
    out, _ = orc.onco_step(s, p, n)
    assert np.array_equal(out["vol"], s["vol"] + 42.0)      # V += growth exactly
    want_d = 2.0 * np.cbrt(out["vol"] * (0.75 / math.pi))
    assert np.all(np.abs(out["d"] - want_d) <= 4e-16 * want_d)
    assert np.all(out["flags"] & orc.GREW)


def test_certain_division_and_fresh_ids():
    n = 3000
    s = _pop(n, d=14.0)
    p = orc.onco_params(max_diameter=14.0, p_death=0.0, p_div=1.0, displacement_rate=0.0, step=4)
    out, nxt = orc.onco_step(s, p, 10_000)
    assert len(out["x"]) == 2 * n and nxt == 10_000 + n
    mothers, daughters = slice(0, n), slice(n, 2 * n)
    assert np.array_equal(out["id"][mothers], s["id"])
    assert np.array_equal(out["id"][daughters], np.arange(10_000, 10_000 + n))  # mother-id order
    assert np.array_equal(out["vol"][mothers] + out["vol"][daughters], s["vol"])  # V/2 + V/2
    assert np.array_equal(out["vol"][mothers], out["vol"][daughters])
    gap = np.sqrt(sum((out[c][mothers] - out[c][daughters]) ** 2 for c in ("x", "y", "z")))
    assert np.all(np.abs(gap - out["d"][mothers]) <= 1e-12 * out["d"][mothers])  # touching
    assert np.all(out["flags"][daughters] == orc.ADDED)
    assert np.all(out["age"][daughters] == 0)
    assert len(np.unique(out["id"])) == 2 * n


def test_division_frequency_and_accounting():
    n = 30000
    s = _pop(n, d=14.0, ages=np.full(n, 100))
    p = orc.onco_params(max_diameter=14.0, p_death=0.1, p_div=0.3, step=9)
    out, nxt = orc.onco_step(s, p, n)
    ndiv = nxt - n
    # a division draw only for survivors: E[div] = n (1 - p_death) p_div
    mu = n * 0.9 * 0.3
    assert abs(ndiv - mu) < 5 * math.sqrt(n * 0.27 * 0.73)
    nsurv = len(out["x"]) - ndiv
    assert abs((n - nsurv) - 0.1 * n) < 5 * math.sqrt(n * 0.09)
    assert len(np.unique(out["id"])) == len(out["id"])
    # survivors keep their data except position / volume / diameter / flags / age
    surv = out["id"][:nsurv]
    idx = np.searchsorted(s["id"], surv)
    assert np.array_equal(s["id"][idx], surv)
    assert np.all(np.diff(idx) > 0)                       # order kept


@pytest.mark.parametrize("max_age", [1, 120])
def test_initial_ages_in_range(max_age):
    a = orc.init_ages(np.arange(10000, dtype=np.uint32), 1, max_age)
    assert a.min() >= 0 and a.max() < max_age
    if max_age > 1:
        assert abs(a.mean() - (max_age - 1) / 2) < 5 * max_age / math.sqrt(12 * 10000)
