"""Pins of the oracle's diffusion / secretion / chemotaxis against
what the mathematics and the paper fix -- none of them re-evaluates the oracle's formula:

* discrete sine eigenmodes: with zero values outside the grid (R34) the product of sine
  modes sin(pi a (i+1)/(nx+1)) ... is an eigenvector of the explicit scheme of Eq. 4.3
  with eigenvalue lambda = (1 - mu dt) + sum_d c_d (2 cos(pi a_d/(n_d+1)) - 2), so n steps
  multiply it by lambda^n (closed form; pins the coefficients, the axis mapping, the
  boundary and the decay);
* decay only (nu = 0): every stencil term vanishes exactly;
* mass conservation (mu = 0, mass far from the boundary);
* convergence to the heat kernel M/(4 pi nu t)^{3/2} exp(-r^2/(4 nu t)) at r = sqrt(1000)
  um from an instantaneous point source as the resolution increases (the paper's own
  diffusion convergence test);
* secretion and chemotaxis closed forms (k agents in one cell; linear fields).
"""
import math

import numpy as np
import pytest

import oracle as orc


def _mode(g, a, b, c):
    i = np.arange(g.nx)
    j = np.arange(g.ny)
    k = np.arange(g.nz)
    sx = np.sin(math.pi * a * (i + 1) / (g.nx + 1))
    sy = np.sin(math.pi * b * (j + 1) / (g.ny + 1))
    sz = np.sin(math.pi * c * (k + 1) / (g.nz + 1))
    return sz[:, None, None] * sy[None, :, None] * sx[None, None, :]


def _lambda(g, nu, mu, dt, a, b, c):
    cx, cy, cz = nu * dt / g.dx ** 2, nu * dt / g.dy ** 2, nu * dt / g.dz ** 2
    return ((1 - mu * dt) + cx * (2 * math.cos(math.pi * a / (g.nx + 1)) - 2)
            + cy * (2 * math.cos(math.pi * b / (g.ny + 1)) - 2)
            + cz * (2 * math.cos(math.pi * c / (g.nz + 1)) - 2))


@pytest.mark.parametrize("modes", [[(2, 3, 1)], [(1, 1, 1), (4, 2, 5)]])
def test_sine_eigenmodes(modes):
    g = orc.Grid3(13, 9, 7, dx=1.5, dy=0.8, dz=2.1)
    nu, mu, dt, n = 0.3, 0.05, 0.5, 20
    u0 = sum(_mode(g, *m) for m in modes)
    want = sum(_lambda(g, nu, mu, dt, *m) ** n * _mode(g, *m) for m in modes)
    got = orc.diffuse(u0, g, nu, mu, dt, n)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(u0))


def test_decay_only_is_exact():
    g = orc.Grid3(6, 5, 4, dx=1.0)
    rng = np.random.default_rng(3)
    u0 = rng.uniform(0, 10, (4, 5, 6))
    mu, dt = 0.02, 0.7
    d = 1.0 - mu * dt
    want = u0.copy()
    for _ in range(9):
        want = want * d
    got = orc.diffuse(u0, g, 0.0, mu, dt, 9)
    assert np.array_equal(got, want)


def test_mass_conservation_without_decay():
    g = orc.Grid3(40, 36, 32, dx=1.0)
    z, y, x = np.meshgrid(np.arange(32), np.arange(36), np.arange(40), indexing="ij")
    # variance 1 -> 1 + 2 nu t = 3 after 10 steps; the boundary stays > 9 sigma away
    u0 = np.exp(-((x - 20) ** 2 + (y - 18) ** 2 + (z - 16) ** 2) / 2.0)
    got = orc.diffuse(u0, g, 1.0, 0.0, 0.1, 10)
    assert abs(got.sum() - u0.sum()) <= 1e-12 * u0.sum()
    assert got.max() < u0.max()          # it spreads
    assert got.min() >= 0.0


def _probe_error(delta):
    """Max relative error of the grid value against the heat kernel at the probe
    (30, 10, 0) um = sqrt(1000) um from a unit point source, t in [100, 300] s."""
    nu, m = 1.0, 1.0
    n = int(round(125.0 / delta)) | 1             # odd: the source sits on the centre cell
    g = orc.Grid3(n, n, n, dx=delta)
    c = n // 2
    u = np.zeros((n, n, n))
    u[c, c, c] = m / delta ** 3
    dt = 0.9 * delta ** 2 / (6 * nu)
    pi, pj = c + int(round(30 / delta)), c + int(round(10 / delta))
    err, t = 0.0, 0.0
    for step in range(int(300 / dt) + 1):
        if t >= 100.0:
            exact = m / (4 * math.pi * nu * t) ** 1.5 * math.exp(-1000.0 / (4 * nu * t))
            err = max(err, abs(u[c, pj, pi] - exact) / exact)
        u = orc.diffuse(u, g, nu, 0.0, dt, 1)
        t += dt
    return err


def test_converges_to_heat_kernel_at_sqrt1000():
    e_coarse, e_fine = _probe_error(5.0), _probe_error(2.5)
    assert e_fine < 0.5 * e_coarse        # second order in space and time: ~4x
    assert e_fine < 0.05


def test_secretion_closed_form():
    g = orc.Grid3(4, 5, 6, lo=(10.0, -5.0, 0.0), dx=2.0, dy=1.0, dz=3.0)
    # cell (1, 2, 3): x in [12, 14), y in [-3, -2), z in [9, 12)
    pts = [(12.0, -3.0, 9.0), (13.9, -2.5, 11.9), (12.5, -2.01, 10.0),   # 3 agents, cell (1,2,3)
           (0.0, -50.0, -1.0), (10.5, -4.5, 2.0),                         # 2 agents, cell (0,0,0)
           (100.0, 100.0, 100.0),                                         # clamped to the far corner
           (13.0, -2.5, 10.0)]                                            # other type
    s = {"x": np.array([p[0] for p in pts]), "y": np.array([p[1] for p in pts]),
         "z": np.array([p[2] for p in pts])}
    t = np.array([1, 1, 1, 1, 1, 1, 0], np.uint8)
    u = orc.secrete(s, t, 1, 1.0, np.zeros((6, 5, 4)), g)
    want = np.zeros((6, 5, 4))
    want[3, 2, 1] = 3.0
    want[0, 0, 0] = 2.0
    want[5, 4, 3] = 1.0
    assert np.array_equal(u, want)


def test_chemotaxis_linear_fields():
    g = orc.Grid3(8, 8, 8, dx=1.0)
    z, y, x = np.meshgrid(np.arange(8.0), np.arange(8.0), np.arange(8.0), indexing="ij")
    s = {"x": np.array([3.5, 0.5, 4.2]), "y": np.array([3.5, 2.5, 4.9]),
         "z": np.array([3.5, 6.5, 1.1])}
    t = np.zeros(3, np.uint8)
    # u = 3 i: the central difference is exactly 3 (interior) and 1.5 at the i = 0 edge
    # (outside = 0); either way the normalized gradient is +x
    out = orc.chemotaxis(s, t, 0, 0.75, 3.0 * x, g)
    assert np.array_equal(out["x"], s["x"] + 0.75)
    assert np.array_equal(out["y"], s["y"]) and np.array_equal(out["z"], s["z"])
    # u = i + 2 j + 2 k (interior cells): gradient (1, 2, 2), norm 3
    out = orc.chemotaxis(s, t, 0, 0.75, x + 2 * y + 2 * z, g)
    k = [0, 2]   # agents 0 and 2 sit in interior cells
    assert np.array_equal(out["x"][k], s["x"][k] + 0.75 * (1 / 3))
    assert np.array_equal(out["y"][k], s["y"][k] + 0.75 * (2 / 3))
    assert np.array_equal(out["z"][k], s["z"][k] + 0.75 * (2 / 3))
    # constant field: zero gradient inside (no move); at an edge cell the zero outside
    # (R34) makes the gradient point inwards: agent 1 (cell i = 0) moves +x by 0.75
    out = orc.chemotaxis(s, t, 0, 0.75, np.full((8, 8, 8), 4.0), g)
    for c in ("x", "y", "z"):
        assert np.array_equal(out[c][k], s[c][k])
    assert out["x"][1] == s["x"][1] + 0.75
    assert out["y"][1] == s["y"][1] and out["z"][1] == s["z"][1]
