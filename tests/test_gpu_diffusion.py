"""GPU parity for extracellular diffusion, secretion and chemotaxis
through the C ABI, against the pinned oracle (tests/test_oracle_diffusion.py).

Bit-exact: Eq. 4.3 in the operation order of reading R35 (no fused multiply-add on
either side), secretion (every addend is the same q, so the atomic order does not
matter), chemotaxis (R37, R38).
"""
import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_10796_b200 import Engine
    e = Engine(0, 1 << 12)
    yield e
    e.close()


def _grids(nx, ny, nz, lo, dx, dy, dz):
    from paper_2503_10796_b200 import CGrid3
    return CGrid3.make(nx, ny, nz, lo, dx, dy, dz), orc.Grid3(nx, ny, nz, lo, dx, dy, dz)


@pytest.mark.parametrize("shape,steps", [
    ((1, 1, 1), 3),
    ((33, 17, 5), 4),        # ragged against the 32 x 16 tile
    ((64, 48, 130), 3),      # crosses a 128-plane z chunk; odd step count
    ((37, 70, 260), 2),      # several z chunks
    ((5, 3, 301), 1),
])
def test_diffuse_bit_exact(eng, shape, steps):
    import torch
    nx, ny, nz = shape
    rng = np.random.default_rng(nx * 1000 + nz)
    u0 = rng.uniform(0.0, 5.0, (nz, ny, nx))
    cg, og = _grids(nx, ny, nz, (0.0, 0.0, 0.0), 1.3, 0.9, 1.7)
    nu, mu, dt = 0.2, 0.03, 0.6
    u = torch.from_numpy(u0).cuda()
    v = torch.empty_like(u)
    for _ in range(steps):
        eng.diffuse(u, v, cg, nu, mu, dt)
        u, v = v, u
    torch.cuda.synchronize()
    want = orc.diffuse(u0, og, nu, mu, dt, steps)
    assert np.array_equal(u.cpu().numpy(), want)


def test_diffuse_eigenmode_on_gpu(eng):
    """The discrete sine mode decays by its closed-form eigenvalue on the GPU too."""
    import math
    import torch
    nx, ny, nz = 40, 24, 140
    cg, og = _grids(nx, ny, nz, (0.0, 0.0, 0.0), 1.0, 1.0, 1.0)
    i, j, k = np.arange(nx), np.arange(ny), np.arange(nz)
    mode = (np.sin(math.pi * 3 * (k + 1) / (nz + 1))[:, None, None]
            * np.sin(math.pi * (j + 1) / (ny + 1))[None, :, None]
            * np.sin(math.pi * 2 * (i + 1) / (nx + 1))[None, None, :])
    nu, mu, dt, n = 0.15, 0.01, 1.0, 25
    lam = ((1 - mu * dt) + nu * dt * (2 * math.cos(math.pi * 2 / (nx + 1)) - 2)
           + nu * dt * (2 * math.cos(math.pi / (ny + 1)) - 2)
           + nu * dt * (2 * math.cos(math.pi * 3 / (nz + 1)) - 2))
    u = torch.from_numpy(mode).cuda()
    v = torch.empty_like(u)
    for _ in range(n):
        eng.diffuse(u, v, cg, nu, mu, dt)
        u, v = v, u
    got = u.cpu().numpy()
    assert np.max(np.abs(got - lam ** n * mode)) <= 1e-12


def _agents(n, lo, hi, seed):
    from paper_2503_10796_b200 import Agents
    rng = np.random.default_rng(seed)
    s = {c: rng.uniform(lo[i], hi[i], n) for i, c in enumerate(("x", "y", "z"))}
    s["d"] = np.full(n, 10.0)
    s["id"] = np.arange(n, dtype=np.uint32)
    s["flags"] = np.zeros(n, np.uint32)
    return s, Agents.from_numpy(s)


@pytest.mark.parametrize("q", [1.0, 0.3])
def test_secrete_bit_exact(eng, q):
    import torch
    cg, og = _grids(20, 12, 9, (-5.0, 2.0, 0.0), 2.0, 1.5, 3.0)
    # positions partly outside the grid (clamped, R36); many agents per cell
    s, a = _agents(5000, (-10.0, 0.0, -3.0), (40.0, 22.0, 30.0), 7)
    t = np.random.default_rng(8).integers(0, 2, 5000).astype(np.uint8)
    tt = torch.from_numpy(t).cuda()
    u0 = np.random.default_rng(9).uniform(0, 1, (9, 12, 20))
    for sel in (0, 1):
        u = torch.from_numpy(u0).cuda()
        eng.secrete(a, tt, sel, q, u, cg)
        torch.cuda.synchronize()
        assert np.array_equal(u.cpu().numpy(), orc.secrete(s, t, sel, q, u0, og))


def test_chemotaxis_bit_exact(eng):
    import torch
    cg, og = _grids(24, 20, 16, (0.0, 0.0, 0.0), 1.0, 1.25, 0.8)
    s, a = _agents(3000, (-2.0, -2.0, -2.0), (26.0, 27.0, 15.0), 11)
    t = np.random.default_rng(12).integers(0, 2, 3000).astype(np.uint8)
    u0 = np.random.default_rng(13).uniform(0, 1, (16, 20, 24))
    u0[3:6, 4:8, 5:9] = 0.5   # a flat patch: zero gradients inside it
    eng.chemotaxis(a, torch.from_numpy(t).cuda(), 1, 0.75, torch.from_numpy(u0).cuda(), cg)
    torch.cuda.synchronize()
    want = orc.chemotaxis(s, t, 1, 0.75, u0, og)
    g = a.numpy()
    for c in ("x", "y", "z"):
        assert np.array_equal(g[c], want[c]), c


def test_soma_steps_bit_exact(eng):
    """Secretion, chemotaxis and diffusion of two substances over several steps (R39)."""
    import torch
    cg, og = _grids(30, 30, 30, (0.0, 0.0, 0.0), 2.0, 2.0, 2.0)
    s, a = _agents(2000, (0.0, 0.0, 0.0), (60.0, 60.0, 60.0), 21)
    t = np.random.default_rng(22).integers(0, 2, 2000).astype(np.uint8)
    tt = torch.from_numpy(t).cuda()
    grids = [torch.zeros((30, 30, 30), dtype=torch.float64, device="cuda") for _ in range(2)]
    spares = [torch.empty_like(grids[0]) for _ in range(2)]
    og_u = [np.zeros((30, 30, 30)) for _ in range(2)]
    nu, mu, dt, q, w = 0.4, 0.1, 0.5, 1.0, 0.75
    for step in range(4):
        grids, spares = eng.soma_step(a, tt, grids, spares, cg, nu, mu, dt, q, w)
        s, og_u = orc.soma_step(s, t, og_u, og, nu, mu, dt, q, w)
        torch.cuda.synchronize()
        g = a.numpy()
        for c in ("x", "y", "z"):
            assert np.array_equal(g[c], s[c]), (step, c)
        for k in range(2):
            assert np.array_equal(grids[k].cpu().numpy(), og_u[k]), (step, k)


def test_diffuse_full_size_sampled(eng):
    """A 256^3 grid (the bench uses 512^3 per substance; 256^3 keeps the oracle at about
    a second for its 16.8M-point step), one step, compared on every point."""
    import torch
    n = 256
    cg, og = _grids(n, n, n, (0.0, 0.0, 0.0), 2.0, 2.0, 2.0)
    u0 = np.random.default_rng(31).uniform(0.0, 1.0, (n, n, n))
    u = torch.from_numpy(u0).cuda()
    v = torch.empty_like(u)
    eng.diffuse(u, v, cg, 1.0, 0.1, 0.5)
    want = orc.diffuse(u0, og, 1.0, 0.1, 0.5, 1)
    assert np.array_equal(v.cpu().numpy(), want)


@pytest.mark.parametrize("shape", [(64, 48, 130), (34, 18, 3), (2, 1, 129), (96, 40, 257),
                                   (36, 20, 1), (98, 35, 2)])
def test_diffuse_tma_equals_fallback(eng, shape):
    """The TMA-pipelined stencil (nx even) and the register/shared-memory kernel give the
    same bits (and the oracle's), incl. tiles and z chunks cut by the grid edge."""
    import torch
    nx, ny, nz = shape
    u0 = np.random.default_rng(nx + ny + nz).uniform(0.0, 2.0, (nz, ny, nx))
    cg, og = _grids(nx, ny, nz, (0.0, 0.0, 0.0), 0.7, 1.1, 0.9)
    out = []
    for tma in (1, 0):
        eng.set_option("diffuse_tma", tma)
        u = torch.from_numpy(u0).cuda()
        v = torch.empty_like(u)
        for _ in range(3):
            eng.diffuse(u, v, cg, 0.1, 0.02, 0.8)
            u, v = v, u
        out.append(u.cpu().numpy())
    eng.set_option("diffuse_tma", 1)
    assert np.array_equal(out[0], out[1])
    assert np.array_equal(out[0], orc.diffuse(u0, og, 0.1, 0.02, 0.8, 3))
