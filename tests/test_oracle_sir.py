"""Pins for the oracle's SIR step (cfg4; Algorithms 7-9)."""
import math

import numpy as np
import pytest


def test_wrap_worked_examples(orc):
    """Alg. 9: fmod then add max_bound when negative."""
    assert orc.wrap(105.0, 100.0) == 5.0
    assert orc.wrap(-3.0, 100.0) == 97.0
    assert orc.wrap(50.0, 100.0) == 50.0
    assert orc.wrap(100.0, 100.0) == 0.0
    # R20: the literal rule can round to exactly max_bound (box index clamped later)
    assert orc.wrap(-1e-20, 100.0) == 100.0


def _brute_infected_neighbours(s, side, R):
    """Pure-Python min-image recount: S agents with an infected agent within R."""
    X = np.stack([s["x"], s["y"], s["z"]], 1)
    inf = np.nonzero(s["state"] == orc_I)[0]
    sus = np.nonzero(s["state"] == orc_S)[0]
    hit = set()
    for i in sus.tolist():
        for j in inf.tolist():
            d = X[i] - X[j]
            d = np.where(d > side / 2, d - side, np.where(d < -side / 2, d + side, d))
            if float(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) <= R * R:
                hit.add(i)
                break
    return hit


orc_S, orc_I, orc_R = 0, 1, 2


@pytest.mark.parametrize("seed", [1, 2, 3, 17])
def test_infection_set_equals_bruteforce_periodic(orc, seed):
    """p_inf = 1, p_rec = 0: exactly the susceptible agents with an infected agent within
    R (minimum image across the periodic faces) become infected."""
    side, R = 20.0, 2.0
    s = orc.init_sir(600, seed, side, 40)
    want = _brute_infected_neighbours(s, side, R)
    out, counts, ni = orc.sir_step(s, side, R, 1.0, 0.0, seed, 0)
    got = set(np.nonzero((s["state"] == orc_S) & (out["state"] == orc_I))[0].tolist())
    assert got == want
    assert ni == len(want)
    assert counts.sum() == 600 and counts[1] == 40 + len(want)


def test_single_infected_near_corner(orc):
    side, R = 30.0, 2.0
    s = orc.init_sir(2000, 5, side, 0)
    s["x"][0], s["y"][0], s["z"][0] = 0.3, 29.8, 0.1   # corner: neighbours wrap around
    s["state"][0] = orc_I
    # neighbours across each periodic face (inside R only through the minimum image)
    for k, (px, py, pz) in enumerate([(29.5, 29.8, 0.1), (0.3, 0.5, 0.1), (0.3, 29.8, 29.2),
                                      (29.0, 0.9, 29.9), (27.9, 29.8, 0.1)], start=1):
        s["x"][k], s["y"][k], s["z"][k] = px, py, pz
    want = _brute_infected_neighbours(s, side, R)
    out, _, _ = orc.sir_step(s, side, R, 1.0, 0.0, 5, 3)
    got = set(np.nonzero((s["state"] == orc_S) & (out["state"] == orc_I))[0].tolist())
    assert got == want and len(want) > 0


def test_conservation_and_recovery(orc):
    side = 60.0
    s = orc.init_sir(20000, 1, side, 2000)
    for t in range(5):
        s, counts, _ = orc.sir_step(s, side, 2.0, 0.1, 0.01, 1, t)
        assert counts.sum() == 20000
        assert np.array_equal(counts, np.bincount(s["state"], minlength=3))
    # p_rec = 1: every infected agent (old or new) recovers within the step (R18)
    s2, counts, _ = orc.sir_step(s, side, 2.0, 0.5, 1.0, 1, 9)
    assert counts[1] == 0 and np.all(s2["state"][s["state"] == orc_R] == orc_R)


def test_recovery_fraction_binomial(orc):
    side = 500.0
    s = orc.init_sir(200000, 3, side, 200000)        # everyone infected
    out, counts, _ = orc.sir_step(s, side, 2.0, 0.0, 0.01, 3, 0)
    sd = math.sqrt(200000 * 0.01 * 0.99)
    assert abs(counts[2] - 2000) < 5 * sd


def test_movement_closed_forms(orc):
    """v = 2u - 1 capped at |v| = 1 (R16): E|v|^2 = pi/10 + 1 - pi/6 = 0.790560...,
    E|v| = pi/8 + 1 - pi/6 = 0.869100...; |step| <= 1 (min image)."""
    side = 1000.0
    n = 400000
    s = orc.init_sir(n, 7, side, 0)
    out, _, _ = orc.sir_step(s, side, 2.0, 0.0, 0.0, 7, 11)
    d = np.stack([out["x"] - s["x"], out["y"] - s["y"], out["z"] - s["z"]], 1)
    d = np.where(d > side / 2, d - side, np.where(d < -side / 2, d + side, d))
    r2 = (d * d).sum(1)
    r = np.sqrt(r2)
    assert r.max() <= 1.0 + 1e-12
    e2 = math.pi / 10 + 1 - math.pi / 6
    e1 = math.pi / 8 + 1 - math.pi / 6
    assert abs(r2.mean() - e2) < 5 * r2.std() / math.sqrt(n)
    assert abs(r.mean() - e1) < 5 * r.std() / math.sqrt(n)
    assert np.all((out["x"] >= 0) & (out["x"] <= side))


def test_infection_probability(orc):
    """Every susceptible agent sits next to an infected one; p_inf = 0.3 infects ~30 %."""
    side, R = 400.0, 2.0
    n = 40000
    s = orc.init_sir(n, 11, side, 0)
    pairs = n // 2
    s["x"][1::2] = s["x"][0::2] + 0.5                 # partner 0.5 m away (inside R)
    s["x"] = np.mod(s["x"], side)
    s["y"][1::2] = s["y"][0::2]
    s["z"][1::2] = s["z"][0::2]
    s["state"][0::2] = orc_I
    out, counts, ni = orc.sir_step(s, side, R, 0.3, 0.0, 11, 0)
    sd = math.sqrt(pairs * 0.3 * 0.7)
    assert abs(ni - 0.3 * pairs) < 5 * sd
