"""CPU oracle for the BioDynaMo/TeraAgent mechanics hot path (arXiv 2503.10796).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this package.
The product package ``paper_2503_10796_b200`` never imports it and shares no code
with it.

The arithmetic lives in plain C (``oracle/oracle.c``; fp64, ``-ffp-contract=off``,
explicit ``fma`` at the two canonical sites).  This module only marshals numpy
arrays through ctypes.  Each function cites the passage of PAPER.md it follows in
the C source.

Parity status per function (DESIGN.md section 4 lists the pins):
  philox4x32_10        pinned (ATen's philox_engine, a library routine)
  init_spheres         pinned (exact u53 mapping, moments)
  neighbor_pairs_*     pinned (brute force on tiny inputs, pure-Python recount)
  mech_step            pinned (Eq. 4.1 closed forms, antisymmetry, cap, static transparency)
  sorted_order         pinned (Morton worked example P:4762-4766, sortedness invariants)
  diffuse_step         pinned (discrete sine eigenmodes, decay-only, mass conservation,
                       convergence to the heat kernel at sqrt(1000) um)
  secrete, chemotaxis  pinned (closed forms: k agents per cell, linear fields)
  lz4_*, aura_*        pinned (LZ4 block-format streams built by hand from the format
                       definition, round trips, worst-case expansion bound, zero runs;
                       delta encoding: XOR identities, placeholders, new agents, the
                       reference-order defragmentation of P:6350-6352)
  onco_step            pinned (unit Brownian steps, exact age/volume bookkeeping, the
                       age gate, death / division frequencies within 5 sigma, removal
                       invariants, id uniqueness, population accounting)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "oracle.c")]

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

MOVED, GREW, ADDED, STATIC = 1, 2, 4, 8
NNZ_SHIFT = 4


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no CUDA)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + ".tmp"
        subprocess.check_call(["gcc", *CFLAGS, *_SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        u64 = ctypes.c_uint64
        dbl = ctypes.c_double
        i32 = ctypes.c_int
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_u53.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.orc_u53.restype = dbl
        L.orc_u32.argtypes = [ctypes.c_uint32]
        L.orc_u32.restype = dbl
        L.orc_init_spheres.argtypes = [i64, i64, u64, dbl, dbl, dbl, i32, P, P, P, P, P, P]
        L.orc_morton.argtypes = [P, i32, i32]
        L.orc_morton.restype = u64
        L.orc_blocked_key.argtypes = [i64, i64, i64, P]
        L.orc_blocked_key.restype = u64
        L.orc_grid_geometry.argtypes = [i64, P, P, P, P, dbl, P, P, P, P]
        L.orc_neighbor_pairs_brute.argtypes = [i64, P, P, P, P, dbl, P, i64]
        L.orc_neighbor_pairs_brute.restype = i64
        L.orc_neighbor_pairs_grid.argtypes = [i64, P, P, P, P, P, dbl, P, i64]
        L.orc_neighbor_pairs_grid.restype = i64
        L.orc_pair_force.argtypes = [dbl, dbl, dbl, dbl, dbl, P, P]
        L.orc_pair_force.restype = dbl
        L.orc_mech_step.argtypes = [i64, P, P, P, P, P, P, P, i64, P, P, P, P, P, P, P]
        L.orc_sorted_order.argtypes = [i64, P, P, P, P, P, dbl, P, P]
        L.orc_sorted_order_torus.argtypes = [i64, P, P, P, P, P, dbl, dbl, P, P]
        L.orc_cbrt_det.argtypes = [dbl]
        L.orc_cbrt_det.restype = dbl
        L.orc_division_axis.argtypes = [u64, u64, ctypes.c_uint32, P]
        L.orc_grow_divide.argtypes = [i64, P, P, P, P, P, P, P, i64, dbl, dbl, u64, ctypes.c_uint32]
        L.orc_grow_divide.restype = i64
        L.orc_wrap.argtypes = [dbl, dbl]
        L.orc_wrap.restype = dbl
        L.orc_sir_step.argtypes = [i64, P, P, P, P, P, dbl, dbl, dbl, dbl, u64, ctypes.c_uint32, P]
        L.orc_sir_step.restype = i64
        L.orc_init_sir.argtypes = [i64, u64, dbl, i64, P, P, P, P, P]
        L.orc_sir_step_sample.argtypes = [i64, P, P, P, P, P, dbl, dbl, dbl, dbl, u64,
                                          ctypes.c_uint32, i64, P, P, P, P, P, P]
        L.orc_sir_step_sample.restype = i64
        L.orc_diffuse_step.argtypes = [i64, i64, i64, P, P, dbl, dbl, dbl, dbl, dbl, dbl]
        L.orc_onco_step.argtypes = [i64, P, P, P, P, P, P, P, P, i64, P, P]
        L.orc_onco_step.restype = i64
        L.orc_init_ages.argtypes = [i64, P, u64, ctypes.c_uint32, P]
        L.orc_secrete.argtypes = [i64, P, P, P, P, i32, dbl, P, i64, i64, i64, P, dbl, dbl, dbl]
        L.orc_chemotaxis.argtypes = [i64, P, P, P, P, i32, dbl, P, i64, i64, i64, P, dbl, dbl, dbl]
        u8p = P
        L.orc_lz4_compress_block.argtypes = [u8p, i64, u8p, i64]
        L.orc_lz4_compress_block.restype = i64
        L.orc_lz4_decompress_block.argtypes = [u8p, i64, u8p, i64]
        L.orc_lz4_decompress_block.restype = i64
        L.orc_aura_payload_size.argtypes = [i64, i64]
        L.orc_aura_payload_size.restype = i64
        L.orc_aura_payload.argtypes = [i64, P, P, P, P, P, P, i64, P, P, P, P, P, P, P, P]
        L.orc_aura_payload.restype = i64
        L.orc_aura_unpayload.argtypes = [P, i64, i64, P, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_aura_unpayload.restype = i64
        L.orc_aura_compress.argtypes = [P, i64, i64, i64, P, i64]
        L.orc_aura_compress.restype = i64
        L.orc_aura_decompress.argtypes = [P, i64, P, i64, P, P]
        L.orc_aura_decompress.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class MechParams(ctypes.Structure):
    """Mirror of ``orc_mech_params`` (oracle.c)."""

    _fields_ = [
        ("k", ctypes.c_double),
        ("gamma", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("max_disp", ctypes.c_double),
        ("force_threshold", ctypes.c_double),
        ("radius", ctypes.c_double),
        ("detect_static", ctypes.c_int32),
        ("boundary", ctypes.c_int32),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("use_frame", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("frame", ctypes.c_double * 4),
    ]


class Counters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("cand", "nbr", "cont", "n_static")]


def mech_params(k=2.0, gamma=1.0, dt=0.01, max_disp=3.0, force_threshold=0.0, radius=0.0,
                detect_static=False, boundary=0, lo=(0.0, 0.0, 0.0), hi=(0.0, 0.0, 0.0),
                frame=None):
    """frame: optional global grid frame (o_x, o_y, o_z, R) of a partitioned run."""
    p = MechParams()
    if frame is not None:
        p.use_frame = 1
        p.frame[:] = [float(v) for v in frame]
    p.k, p.gamma, p.dt, p.max_disp = k, gamma, dt, max_disp
    p.force_threshold, p.radius = force_threshold, radius
    p.detect_static, p.boundary = int(bool(detect_static)), int(boundary)
    p.lo[:] = list(lo)
    p.hi[:] = list(hi)
    return p


# ----------------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def u53(wa: int, wb: int) -> float:
    return lib().orc_u53(wa, wb)


def u32(w: int) -> float:
    return lib().orc_u32(w)


def init_spheres(n, seed, side, d_lo, d_width=0.0, d_random=False, id0=0):
    """Uniform-in-cube population, per-id Philox (R22/R23/R29).

    Returns dict of numpy arrays x, y, z, d (f64), id, flags (u32)."""
    s = {k: np.zeros(n, np.float64) for k in ("x", "y", "z", "d")}
    s["id"] = np.zeros(n, np.uint32)
    s["flags"] = np.zeros(n, np.uint32)
    lib().orc_init_spheres(id0, n, seed, side, d_lo, d_width, int(bool(d_random)),
                           _p(s["x"]), _p(s["y"]), _p(s["z"]), _p(s["d"]),
                           _p(s["id"]), _p(s["flags"]))
    return s


def morton(coords, bits) -> int:
    c = np.asarray(coords, dtype=np.uint32)
    return int(lib().orc_morton(_p(c), len(c), bits))


def blocked_key(bx, by, bz, D) -> int:
    Da = np.asarray(D, dtype=np.int64)
    return int(lib().orc_blocked_key(bx, by, bz, _p(Da)))


def grid_geometry(s, radius=0.0):
    n = len(s["x"])
    R = ctypes.c_double()
    L = ctypes.c_double()
    o = np.zeros(3, np.float64)
    D = np.zeros(3, np.int64)
    lib().orc_grid_geometry(n, _p(_f64(s["x"])), _p(_f64(s["y"])), _p(_f64(s["z"])),
                            _p(_f64(s["d"])), radius, ctypes.byref(R), ctypes.byref(L),
                            _p(o), _p(D))
    return R.value, L.value, o, D


def neighbor_pairs_brute(s, R) -> np.ndarray:
    x, y, z, i = _f64(s["x"]), _f64(s["y"]), _f64(s["z"]), _u32(s["id"])
    n = len(x)
    cnt = lib().orc_neighbor_pairs_brute(n, _p(x), _p(y), _p(z), _p(i), R, None, 0)
    out = np.zeros(max(cnt, 1), np.uint64)
    lib().orc_neighbor_pairs_brute(n, _p(x), _p(y), _p(z), _p(i), R, _p(out), cnt)
    return np.sort(out[:cnt])


def neighbor_pairs_grid(s, radius=0.0) -> np.ndarray:
    x, y, z, d, i = (_f64(s["x"]), _f64(s["y"]), _f64(s["z"]), _f64(s["d"]),
                     _u32(s["id"]))
    n = len(x)
    cnt = lib().orc_neighbor_pairs_grid(n, _p(x), _p(y), _p(z), _p(d), _p(i), radius, None, 0)
    out = np.zeros(max(cnt, 1), np.uint64)
    lib().orc_neighbor_pairs_grid(n, _p(x), _p(y), _p(z), _p(d), _p(i), radius, _p(out), cnt)
    return np.sort(out[:cnt])


def pair_force(k, gamma, D, ri, rj):
    """Eq. 4.1/4.2 for one pair at squared distance D: returns (F_N, s, contact)."""
    c = ctypes.c_int()
    sc = ctypes.c_double()
    Fn = lib().orc_pair_force(k, gamma, D, ri, rj, ctypes.byref(c), ctypes.byref(sc))
    return Fn, sc.value, bool(c.value)


def mech_step(s, params: MechParams, sample=None):
    """One mechanics step (copy semantics).  Returns (out, counters).

    out holds x, y, z, flags and the summed force (m x 3; zero for static agents) for
    every agent (input order) or for the agents listed in
    ``sample`` (in that order); d and id are unchanged by a mechanics step."""
    x, y, z, d = _f64(s["x"]), _f64(s["y"]), _f64(s["z"]), _f64(s["d"])
    i, f = _u32(s["id"]), _u32(s["flags"])
    n = len(x)
    if sample is None:
        m, idx = n, None
    else:
        idx = np.ascontiguousarray(sample, dtype=np.int64)
        m = len(idx)
    out = {k: np.zeros(m, np.float64) for k in ("x", "y", "z")}
    out["flags"] = np.zeros(m, np.uint32)
    out["force"] = np.zeros((m, 3), np.float64)
    c = Counters()
    lib().orc_mech_step(n, _p(x), _p(y), _p(z), _p(d), _p(i), _p(f), ctypes.byref(params), m,
                        None if idx is None else _p(idx), _p(out["x"]), _p(out["y"]),
                        _p(out["z"]), _p(out["flags"]), _p(out["force"]), ctypes.byref(c))
    if c.n_static < 0:
        raise ValueError("toroidal boundary needs lo = 0, a cube hi[0] = hi[1] = hi[2] and at "
                         "least 3 boxes of edge >= R per axis (R52)")
    return out, {k: getattr(c, k) for k in ("cand", "nbr", "cont", "n_static")}


def sorted_order(s, radius=0.0, torus_side=0.0):
    """Input indices in (blocked Morton key, id) order, and the sorted keys
    (torus_side > 0: the toroidal lattice of R52)."""
    x, y, z, d, i = (_f64(s["x"]), _f64(s["y"]), _f64(s["z"]), _f64(s["d"]),
                     _u32(s["id"]))
    n = len(x)
    perm = np.zeros(n, np.int64)
    keys = np.zeros(n, np.uint64)
    if n:
        lib().orc_sorted_order_torus(n, _p(x), _p(y), _p(z), _p(d), _p(i), radius, torus_side,
                                     _p(perm), _p(keys))
    return perm, keys


def step_full(s, params: MechParams):
    """Convenience: one step returning the full new state in the product's output
    order (sorted by the step's grid), as the GPU library leaves it."""
    out, cnt = mech_step(s, params)
    perm, _ = sorted_order(s, params.radius, params.hi[0] if params.boundary == 2 else 0.0)
    new = {
        "x": out["x"][perm], "y": out["y"][perm], "z": out["z"][perm],
        "d": np.asarray(s["d"], np.float64)[perm], "id": np.asarray(s["id"], np.uint32)[perm],
        "flags": out["flags"][perm],
    }
    return new, cnt


# ---------------------------------------------------------------- growth + division (cfg3)
V_MAX_CFG3 = (3.141592653589793 / 6.0) * 1728.0   # (M_PI/6.0)*1728.0: d = 12 um


def cbrt_det(v: float) -> float:
    """R28 deterministic cube root (8 Newton steps from a power-of-two start)."""
    return lib().orc_cbrt_det(v)


def division_axis(seed: int, agent_id: int, step: int) -> np.ndarray:
    u = np.zeros(3, np.float64)
    lib().orc_division_axis(seed, agent_id, step, _p(u))
    return u


def init_volumes(s):
    """V = (M_PI/6.0)*(d*d*d) per agent (R28 companion, exact op order)."""
    d = np.asarray(s["d"], np.float64)
    return (np.pi / 6.0) * (d * d * d)


def grow_divide(s, growth, v_max, seed, step):
    """Growth/division pass (Alg. 4 control flow + Cell::Divide, R13-R15).  s holds x,
    y, z, d, vol, id, flags (post-mechanics); returns a new dict with daughters
    appended at n + rank (rank among dividers in id order)."""
    n = len(s["x"])
    ndiv = int(np.count_nonzero(~(np.asarray(s["vol"]) < v_max)))
    cap = n + ndiv
    out = {}
    for k in ("x", "y", "z", "d", "vol"):
        a = np.zeros(max(cap, 1), np.float64)
        a[:n] = s[k]
        out[k] = a
    for k in ("id", "flags"):
        a = np.zeros(max(cap, 1), np.uint32)
        a[:n] = s[k]
        out[k] = a
    r = lib().orc_grow_divide(n, _p(out["x"]), _p(out["y"]), _p(out["z"]), _p(out["d"]),
                              _p(out["vol"]), _p(out["id"]), _p(out["flags"]), cap, growth,
                              v_max, seed, step)
    assert r == cap, (r, cap)
    return {k: v[:cap] for k, v in out.items()}


def cfg3_step(s, params: MechParams, growth, v_max, seed, step):
    """One cfg3 step (R15, R27): mechanics on the snapshot (static skip per params),
    then growth/division at the post-mechanics positions.  Input/output in any order."""
    out, cnt = mech_step(s, params)
    post = {"x": out["x"], "y": out["y"], "z": out["z"], "d": s["d"], "vol": s["vol"],
            "id": s["id"], "flags": out["flags"]}
    return grow_divide(post, growth, v_max, seed, step), cnt


# ---------------------------------------------------------------- SIR epidemiology (cfg4)
S_, I_, R_ = 0, 1, 2


def wrap(el: float, max_bound: float) -> float:
    """Alg. 9 toroidal wrap, literal (R20)."""
    return lib().orc_wrap(el, max_bound)


def init_sir(n, seed, side, n_infected):
    s = {k: np.zeros(n, np.float64) for k in ("x", "y", "z")}
    s["state"] = np.zeros(n, np.uint8)
    s["id"] = np.zeros(n, np.uint32)
    lib().orc_init_sir(n, seed, side, n_infected, _p(s["x"]), _p(s["y"]), _p(s["z"]),
                       _p(s["state"]), _p(s["id"]))
    return s


def sir_step(s, side, radius, p_inf, p_rec, seed, step):
    """Algorithms 7-9 (R16-R20, R22) on a copy of s; returns (new state, counts, new
    infections)."""
    out = {k: np.array(v, copy=True) for k, v in s.items()}
    n = len(out["x"])
    for k in ("x", "y", "z"):
        out[k] = np.ascontiguousarray(out[k], np.float64)
    out["state"] = np.ascontiguousarray(out["state"], np.uint8)
    ids = np.ascontiguousarray(out["id"], np.uint32)
    counts = np.zeros(3, np.int64)
    ni = lib().orc_sir_step(n, _p(out["x"]), _p(out["y"]), _p(out["z"]), _p(out["state"]),
                            _p(ids), side, radius, p_inf, p_rec, seed, step, _p(counts))
    return out, counts, ni


def sir_step_sample(s, side, radius, p_inf, p_rec, seed, step, sample):
    """SIR step for the listed agents only (full snapshot for the infected index)."""
    x, y, z = _f64(s["x"]), _f64(s["y"]), _f64(s["z"])
    st = np.ascontiguousarray(s["state"], np.uint8)
    ids = _u32(s["id"])
    idx = np.ascontiguousarray(sample, np.int64)
    m = len(idx)
    out = {k: np.zeros(m, np.float64) for k in ("x", "y", "z")}
    out["state"] = np.zeros(m, np.uint8)
    counts = np.zeros(3, np.int64)
    ni = lib().orc_sir_step_sample(len(x), _p(x), _p(y), _p(z), _p(st), _p(ids), side, radius,
                                   p_inf, p_rec, seed, step, m, _p(idx), _p(out["x"]),
                                   _p(out["y"]), _p(out["z"]), _p(out["state"]), _p(counts))
    return out, counts, ni


# ------------------------------------------------------------------ diffusion (row f4)
class Grid3:
    """Diffusion grid (reading R34): shape (nz, ny, nx) of cell-centred points, the cell
    (i, j, k) being [lo + i d, lo + (i+1) d) per axis; values outside are 0."""

    def __init__(self, nx, ny, nz, lo=(0.0, 0.0, 0.0), dx=1.0, dy=None, dz=None):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.lo = np.ascontiguousarray(lo, np.float64)
        self.dx = float(dx)
        self.dy = float(dx if dy is None else dy)
        self.dz = float(dx if dz is None else dz)


def diffuse(u, g, nu, mu, dt, steps=1):
    """Eq. 4.3, `steps` explicit steps of the (nz, ny, nx) array u (R35)."""
    a = np.ascontiguousarray(u, np.float64).copy()
    b = np.empty_like(a)
    for _ in range(steps):
        lib().orc_diffuse_step(g.nx, g.ny, g.nz, _p(a), _p(b), nu, mu, dt, g.dx, g.dy, g.dz)
        a, b = b, a
    return a


def secrete(s, type_, type_sel, q, u, g):
    """Alg. secretion_module into a copy of u (R36)."""
    out = np.ascontiguousarray(u, np.float64).copy()
    x, y, z = _f64(s["x"]), _f64(s["y"]), _f64(s["z"])
    t = np.ascontiguousarray(type_, np.uint8)
    lib().orc_secrete(len(x), _p(x), _p(y), _p(z), _p(t), int(type_sel), q, _p(out), g.nx, g.ny,
                      g.nz, _p(g.lo), g.dx, g.dy, g.dz)
    return out


def chemotaxis(s, type_, type_sel, weight, u, g):
    """Alg. chemotaxis_module on a copy of the positions (R37, R38)."""
    out = {k: np.array(v, copy=True) for k, v in s.items()}
    for k in ("x", "y", "z"):
        out[k] = np.ascontiguousarray(out[k], np.float64)
    t = np.ascontiguousarray(type_, np.uint8)
    uu = np.ascontiguousarray(u, np.float64)
    lib().orc_chemotaxis(len(out["x"]), _p(out["x"]), _p(out["y"]), _p(out["z"]), _p(t),
                         int(type_sel), weight, _p(uu), g.nx, g.ny, g.nz, _p(g.lo), g.dx, g.dy,
                         g.dz)
    return out


def soma_step(s, type_, grids, g, nu, mu, dt, q, weight):
    """One soma-clustering step (reading R39): secretion of every type into
    its own substance, chemotaxis of every type up its substance's gradient, then one
    diffusion step (Eq. 4.3) of every substance.  Returns (new positions, new grids)."""
    gs = [secrete(s, type_, t, q, grids[t], g) for t in range(len(grids))]
    out = dict(s)
    for t in range(len(grids)):
        out = chemotaxis(out, type_, t, weight, gs[t], g)
    gs = [diffuse(u, g, nu, mu, dt, 1) for u in gs]
    return out, gs


# ------------------------------------------------------------------ oncology (row f2)
class OncoParams(ctypes.Structure):
    """Mirror of orc_onco_params (oracle.c): Alg. 4 with Table 4.2's parameters."""
    _fields_ = [("displacement_rate", ctypes.c_double), ("growth", ctypes.c_double),
                ("max_diameter", ctypes.c_double), ("p_death", ctypes.c_double),
                ("p_div", ctypes.c_double), ("min_age", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("step", ctypes.c_uint32)]


def onco_params(displacement_rate=0.005, growth=42.0, max_diameter=14.0, p_death=0.033,
                p_div=0.0215, min_age=87, seed=1, step=0) -> OncoParams:
    return OncoParams(displacement_rate, growth, max_diameter, p_death, p_div, min_age, seed,
                      step)


def init_ages(ids, seed, max_age):
    """Initial ages (reading R44): floor(u32 * max_age) from Philox (id, 0xFFFFFFFC, 2)."""
    ids = _u32(ids)
    out = np.zeros(len(ids), np.uint32)
    lib().orc_init_ages(len(ids), _p(ids), seed, max_age, _p(out))
    return out


def onco_step(s, p: OncoParams, id_next: int):
    """Alg. 4 + removal (R41-R45) on a copy of s (x, y, z, d, vol, id, flags, age, all
    post-mechanics); returns (new state, new id_next)."""
    n = len(s["x"])
    cap = 2 * n + 1
    out = {}
    for k in ("x", "y", "z", "d", "vol"):
        a = np.zeros(cap, np.float64)
        a[:n] = s[k]
        out[k] = a
    for k in ("id", "flags", "age"):
        a = np.zeros(cap, np.uint32)
        a[:n] = s[k]
        out[k] = a
    nxt = ctypes.c_int64(int(id_next))
    r = lib().orc_onco_step(n, _p(out["x"]), _p(out["y"]), _p(out["z"]), _p(out["d"]),
                            _p(out["vol"]), _p(out["id"]), _p(out["flags"]), _p(out["age"]),
                            cap, ctypes.byref(p), ctypes.byref(nxt))
    assert r >= 0, r
    return {k: v[:r] for k, v in out.items()}, int(nxt.value)


def onco_full_step(s, mp: MechParams, p: OncoParams, id_next: int):
    """One oncology step (R40): mechanics on the snapshot, then Alg. 4 + removal at the
    post-mechanics state.  s carries x, y, z, d, vol, id, flags, age in any order; the
    mechanics leaves the grid's (box, id) order, then removal keeps it and daughters
    follow.  Returns (new state, mechanics counters, new id_next)."""
    out, cnt = mech_step(s, mp)
    perm, _ = sorted_order(s, mp.radius)
    post = {"x": out["x"][perm], "y": out["y"][perm], "z": out["z"][perm],
            "d": np.asarray(s["d"], np.float64)[perm], "id": np.asarray(s["id"], np.uint32)[perm],
            "flags": out["flags"][perm], "vol": np.asarray(s["vol"], np.float64)[perm],
            "age": np.asarray(s["age"], np.uint32)[perm]}
    new, nxt = onco_step(post, p, id_next)
    return new, cnt, nxt


# ---------------------------------------------------------------- row f3 (R46-R51)
AURA_FIELDS = ("x", "y", "z", "d", "id", "flags")
LZ4_CHUNK = 1024  # payload bytes per LZ4 block (R50; ORC_LZ4_CHUNK in oracle.c)


def lz4_compress_block(data: bytes) -> bytes:
    """R50 greedy LZ4 block of data (<= 65535 bytes)."""
    src = np.frombuffer(bytes(data), np.uint8).copy()
    cap = len(src) + len(src) // 255 + 16
    dst = np.zeros(cap, np.uint8)
    k = lib().orc_lz4_compress_block(_p(src), len(src), _p(dst), cap)
    assert k >= 0
    return dst[:k].tobytes()


def lz4_decompress_block(data: bytes, cap: int) -> bytes:
    """LZ4 block decoder; raises ValueError on a malformed block."""
    src = np.frombuffer(bytes(data), np.uint8).copy()
    dst = np.zeros(max(cap, 1), np.uint8)
    k = lib().orc_lz4_decompress_block(_p(src), len(src), _p(dst), cap)
    if k < 0:
        raise ValueError("malformed LZ4 block")
    return dst[:k].tobytes()


def _soa(s):
    return [_f64(s[k]) for k in ("x", "y", "z", "d")] + [_u32(s["id"]), _u32(s["flags"])]


def aura_reference(msg):
    """R46: a reference is a message in ascending id order."""
    o = np.argsort(np.asarray(msg["id"], np.uint32), kind="stable")
    return {k: np.ascontiguousarray(np.asarray(msg[k])[o]) for k in AURA_FIELDS}


def aura_payload(msg, ref):
    """R47-R49: (payload bytes, nnew)."""
    m, r = _soa(msg), _soa(ref)
    n, nref = len(m[0]), len(r[0])
    out = np.zeros(max(lib().orc_aura_payload_size(nref, n), 1), np.uint8)
    nnew = ctypes.c_int64()
    size = lib().orc_aura_payload(n, *[_p(a) for a in m], nref, *[_p(a) for a in r], _p(out),
                                  ctypes.byref(nnew))
    return out[:size].tobytes(), int(nnew.value)


def aura_unpayload(payload: bytes, ref, nnew: int):
    """R51: the message (reference order, then new agents)."""
    r = _soa(ref)
    nref = len(r[0])
    buf = np.frombuffer(bytes(payload), np.uint8).copy()
    cap = nref + nnew
    out = {k: np.zeros(max(cap, 1), np.float64) for k in ("x", "y", "z", "d")}
    out.update({k: np.zeros(max(cap, 1), np.uint32) for k in ("id", "flags")})
    m = lib().orc_aura_unpayload(_p(buf), nref, nnew, *[_p(a) for a in r],
                                 *[_p(out[k]) for k in AURA_FIELDS])
    return {k: v[:m] for k, v in out.items()}


def aura_encode(msg, ref) -> bytes:
    """R46-R50: the compressed stream of msg against ref."""
    payload, nnew = aura_payload(msg, ref)
    src = np.frombuffer(payload, np.uint8).copy() if payload else np.zeros(1, np.uint8)
    size = len(payload)
    cap = 40 + 4 * (size // LZ4_CHUNK + 1) + size + size // 255 + 16 * (size // LZ4_CHUNK + 1) + 16
    out = np.zeros(cap, np.uint8)
    k = lib().orc_aura_compress(_p(src), size, len(ref["id"]), nnew, _p(out), cap)
    assert k >= 0
    return out[:k].tobytes()


def aura_decode(stream: bytes, ref):
    """Inverse of aura_encode (R51)."""
    src = np.frombuffer(bytes(stream), np.uint8).copy()
    cap = max(int(np.frombuffer(src[24:32].tobytes(), np.uint64)[0]) if len(src) >= 32 else 0, 1)
    pay = np.zeros(cap, np.uint8)
    nref, nnew = ctypes.c_int64(), ctypes.c_int64()
    size = lib().orc_aura_decompress(_p(src), len(src), _p(pay), cap, ctypes.byref(nref),
                                     ctypes.byref(nnew))
    if size < 0:
        raise ValueError("malformed aura stream")
    assert nref.value == len(ref["id"])
    return aura_unpayload(pay[:size].tobytes(), ref, int(nnew.value))
