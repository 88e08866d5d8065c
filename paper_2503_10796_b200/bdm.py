"""Thin Python binding of include/bdm.h (libbdm.so, sm_100a).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libbdm.so.  PyTorch provides device memory (CUDA tensors), streams and process
groups.  There is no CPU fallback: if libbdm.so is missing or no GPU is present the
calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbdm.so")

BDM_OK, BDM_EINVAL, BDM_ECAPACITY, BDM_ECUDA, BDM_ENCCL, BDM_ENOTFINITE, BDM_ENOTIMPL = (
    0, -1, -2, -3, -4, -5, -6)
FLAG_MOVED, FLAG_GREW, FLAG_ADDED, FLAG_STATIC = 1, 2, 4, 8
NNZ_SHIFT = 4

# Every symbol include/bdm.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "bdm_create", "bdm_create_ex", "bdm_destroy", "bdm_last_error", "bdm_version", "bdm_init_spheres",
    "bdm_grid_build", "bdm_mech_step", "bdm_step", "bdm_step_host", "bdm_run_host", "bdm_sync",
    "bdm_reserve",
    "bdm_get_stats", "bdm_get_grid_info", "bdm_neighbor_pairs", "bdm_peak_dfma",
    "bdm_selftest_recip_div",
    "bdm_set_option", "bdm_grow_divide", "bdm_sir_step", "bdm_local_frame", "bdm_set_frame",
    "bdm_pack_slab", "bdm_append", "bdm_diffuse", "bdm_secrete", "bdm_chemotaxis",
    "bdm_onco_step", "bdm_tile_curve", "bdm_aura_max_size", "bdm_aura_reference",
    "bdm_aura_encode", "bdm_aura_decode", "bdm_nccl_unique_id", "bdm_dist_init",
    "bdm_aura_exchange", "bdm_dist_init_virtual", "bdm_aura_exchange_virtual", "bdm_aura_pending",
    "bdm_aura_finish",
]
PACK_MIGRATE, PACK_AURA = 1, 2


class BdmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"bdm status {status}: {msg}")
        self.status = status


class CAgents(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("capacity", ctypes.c_int64),
        ("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("z", ctypes.c_void_p),
        ("diameter", ctypes.c_void_p), ("volume", ctypes.c_void_p),
        ("id", ctypes.c_void_p), ("flags", ctypes.c_void_p), ("state", ctypes.c_void_p),
    ]


class CParams(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_double), ("gamma", ctypes.c_double), ("dt", ctypes.c_double),
        ("max_displacement", ctypes.c_double), ("force_threshold", ctypes.c_double),
        ("radius", ctypes.c_double), ("detect_static", ctypes.c_int32),
        ("boundary", ctypes.c_int32), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
        ("seed", ctypes.c_uint64), ("step", ctypes.c_uint32), ("collect_stats", ctypes.c_uint32),
    ]


class CStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("cand", "nbr", "cont", "n_static", "n_moved",
                                              "launches")]


class CGrid3(ctypes.Structure):
    """bdm_grid3: the diffusion grid (R34); u is a (nz, ny, nx) float64 device tensor."""
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("lo", ctypes.c_double * 3), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("dz", ctypes.c_double)]

    @staticmethod
    def make(nx, ny, nz, lo=(0.0, 0.0, 0.0), dx=1.0, dy=None, dz=None) -> "CGrid3":
        g = CGrid3()
        g.nx, g.ny, g.nz = int(nx), int(ny), int(nz)
        g.lo = (ctypes.c_double * 3)(*[float(v) for v in lo])
        g.dx = float(dx)
        g.dy = float(dx if dy is None else dy)
        g.dz = float(dx if dz is None else dz)
        return g


class COncoParams(ctypes.Structure):
    """bdm_onco_params: Alg. 4 with Table 4.2's values per 1 h step (R43: d_max 14 um)."""
    _fields_ = [("displacement_rate", ctypes.c_double), ("growth", ctypes.c_double),
                ("max_diameter", ctypes.c_double), ("p_death", ctypes.c_double),
                ("p_div", ctypes.c_double), ("min_age", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("step", ctypes.c_uint32)]

    @staticmethod
    def make(displacement_rate=0.005, growth=42.0, max_diameter=14.0, p_death=0.033,
             p_div=0.0215, min_age=87, seed=1, step=0) -> "COncoParams":
        return COncoParams(displacement_rate, growth, max_diameter, p_death, p_div, min_age,
                           seed, step)


class CGridInfo(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double), ("L", ctypes.c_double), ("origin", ctypes.c_double * 3),
        ("upper", ctypes.c_double * 3), ("dims", ctypes.c_int64 * 3), ("nslots", ctypes.c_int64),
        ("slot_capacity", ctypes.c_int64),
    ]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen libbdm.so and declare the signatures.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(path)
    P, i64, i32, dbl, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64
    AG = ctypes.POINTER(CAgents)
    PR = ctypes.POINTER(CParams)
    sig = {
        "bdm_create": [ctypes.POINTER(P), ctypes.c_int, i64],
        "bdm_create_ex": [ctypes.POINTER(P), ctypes.c_int, i64, i64, ALLOC_FN, FREE_FN, P],
        "bdm_destroy": [P],
        "bdm_init_spheres": [P, AG, i64, i64, u64, dbl, dbl, dbl, i32, P],
        "bdm_grid_build": [P, AG, AG, dbl, P],
        "bdm_mech_step": [P, AG, PR, P],
        "bdm_step": [P, AG, PR, P],
        "bdm_step_host": [P, AG, AG, AG, PR, P],
        "bdm_run_host": [P, AG, AG, PR, ctypes.c_int32, ctypes.c_int32, P],
        "bdm_sync": [P, P],
        "bdm_reserve": [P, i64, i64],
        "bdm_get_stats": [P, ctypes.POINTER(CStats)],
        "bdm_get_grid_info": [P, ctypes.POINTER(CGridInfo)],
        "bdm_neighbor_pairs": [P, AG, dbl, P, i64, ctypes.POINTER(i64), P],
        "bdm_peak_dfma": [P, ctypes.POINTER(dbl), ctypes.POINTER(i32)],
        "bdm_selftest_recip_div": [P, i64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_ulonglong)],
        "bdm_set_option": [P, ctypes.c_char_p, i64],
        "bdm_grow_divide": [P, AG, PR, dbl, dbl, P, P],
        "bdm_sir_step": [P, AG, PR, dbl, dbl, dbl, dbl, P, P],
        "bdm_local_frame": [P, AG, P, P],
        "bdm_set_frame": [P, P],
        "bdm_pack_slab": [P, AG, dbl, dbl, dbl, i32, AG, AG, P, P],
        "bdm_append": [P, AG, AG, P],
        "bdm_diffuse": [P, P, P, ctypes.POINTER(CGrid3), dbl, dbl, dbl, P],
        "bdm_secrete": [P, AG, P, i32, dbl, P, ctypes.POINTER(CGrid3), P],
        "bdm_chemotaxis": [P, AG, P, i32, dbl, P, ctypes.POINTER(CGrid3), P],
        "bdm_onco_step": [P, AG, P, i64, ctypes.POINTER(COncoParams), i64, P, P],
        "bdm_tile_curve": [i32, P],
        "bdm_aura_reference": [P, AG, AG, P],
        "bdm_aura_encode": [P, AG, AG, P, i64, ctypes.POINTER(i64), P],
        "bdm_aura_decode": [P, P, i64, AG, AG, P],
        "bdm_nccl_unique_id": [P],
        "bdm_dist_init": [P, P, i32, i32, dbl, dbl, dbl],
        "bdm_aura_exchange": [P, AG, AG, P],
        "bdm_dist_init_virtual": [P, i32, P, P, dbl],
        "bdm_aura_exchange_virtual": [P, i32, P, P, P],
        "bdm_aura_pending": [P, P],
        "bdm_aura_finish": [P, AG, AG, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.bdm_aura_max_size.argtypes = [i64, i64]
    L.bdm_aura_max_size.restype = i64
    L.bdm_last_error.restype = ctypes.c_char_p
    L.bdm_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(status: int):
    if status != BDM_OK:
        raise BdmError(status, load_library().bdm_last_error().decode())


def tile_curve(order: int):
    """Host-only (bdm_tile_curve): curve position of each tile x | y<<3 | z<<6 of an
    8^3 super-tile for tile_order `order` (0 row-major, 1 Hilbert), as a list."""
    buf = (ctypes.c_uint16 * 512)()
    _check(load_library().bdm_tile_curve(int(order), ctypes.cast(buf, ctypes.c_void_p)))
    return list(buf)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


@dataclass
class Params:
    """bdm_params.  Defaults: Eq. 4.1 with k = 2, gamma = 1; dt = 0.01 and
    a 3 um cap (BASELINE configs); threshold 0; R = largest diameter."""
    k: float = 2.0
    gamma: float = 1.0
    dt: float = 0.01
    max_displacement: float = 3.0
    force_threshold: float = 0.0
    radius: float = 0.0
    detect_static: bool = False
    boundary: int = 0
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (0.0, 0.0, 0.0)
    seed: int = 1
    step: int = 0
    collect_stats: bool = False

    def c(self) -> CParams:
        p = CParams()
        p.k, p.gamma, p.dt = self.k, self.gamma, self.dt
        p.max_displacement, p.force_threshold, p.radius = (
            self.max_displacement, self.force_threshold, self.radius)
        p.detect_static, p.boundary = int(bool(self.detect_static)), int(self.boundary)
        p.lo[:] = list(self.lo)
        p.hi[:] = list(self.hi)
        p.seed, p.step, p.collect_stats = int(self.seed), int(self.step), int(bool(self.collect_stats))
        return p


@dataclass
class Agents:
    """SoA agent arrays (torch tensors on one device, or pinned host tensors)."""
    x: "object"
    y: "object"
    z: "object"
    diameter: "object"
    id: "object"
    flags: "object"
    n: int = 0
    volume: "object" = None
    state: "object" = None
    _c: CAgents = field(default=None, repr=False)

    @staticmethod
    def empty(capacity: int, device="cuda", pin: bool = False, volume: bool = False,
              state: bool = False) -> "Agents":
        import torch
        kw = dict(device=device) if not pin else dict(pin_memory=True)
        f64 = lambda: torch.empty(capacity, dtype=torch.float64, **kw)  # noqa: E731
        u32 = lambda: torch.empty(capacity, dtype=torch.int32, **kw)    # noqa: E731
        a = Agents(f64(), f64(), f64(), f64(), u32(), u32(), 0)
        if volume:
            a.volume = f64()
        if state:
            a.state = torch.zeros(capacity, dtype=torch.uint8, **kw)
        return a

    @property
    def capacity(self) -> int:
        return int(self.x.numel())

    def grow(self, capacity: int):
        """Reallocate to `capacity` (same device), keeping the first n agents."""
        import torch
        for f in ("x", "y", "z", "diameter", "id", "flags", "volume", "state"):
            t = getattr(self, f)
            if t is None:
                continue
            nt = torch.empty(int(capacity), dtype=t.dtype, device=t.device)
            nt[:self.n].copy_(t[:self.n])
            setattr(self, f, nt)

    def c(self) -> CAgents:
        a = CAgents()
        a.n, a.capacity = int(self.n), self.capacity
        a.x, a.y, a.z, a.diameter = _ptr(self.x), _ptr(self.y), _ptr(self.z), _ptr(self.diameter)
        a.volume, a.id, a.flags, a.state = (_ptr(self.volume), _ptr(self.id), _ptr(self.flags),
                                            _ptr(self.state))
        self._c = a
        return a

    def numpy(self) -> dict:
        """Copy of the live agents as numpy arrays (id/flags as uint32)."""
        import numpy as np
        n = self.n
        out = {k: getattr(self, k)[:n].cpu().numpy() for k in ("x", "y", "z", "diameter")}
        out["d"] = out.pop("diameter")
        if self.id is not None:
            out["id"] = self.id[:n].cpu().numpy().view(np.uint32)
        if self.flags is not None:
            out["flags"] = self.flags[:n].cpu().numpy().view(np.uint32)
        if self.volume is not None:
            out["vol"] = self.volume[:n].cpu().numpy()
        if self.state is not None:
            out["state"] = self.state[:n].cpu().numpy()
        return out

    @staticmethod
    def from_numpy(s: dict, capacity: int = None, device="cuda") -> "Agents":
        import numpy as np
        import torch
        n = len(s["x"])
        cap = max(capacity or n, 1)
        a = Agents.empty(cap, device=device)
        a.n = n
        for k, src in (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "d")):
            getattr(a, k)[:n].copy_(torch.from_numpy(np.ascontiguousarray(s[src], np.float64)))
        a.id[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["id"], np.uint32).view(np.int32)))
        a.flags[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["flags"], np.uint32).view(np.int32)))
        if "vol" in s:
            a.volume = torch.zeros(cap, dtype=torch.float64, device=device)
            a.volume[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["vol"], np.float64)))
        if "state" in s:
            a.state = torch.zeros(cap, dtype=torch.uint8, device=device)
            a.state[:n].copy_(torch.from_numpy(np.ascontiguousarray(s["state"], np.uint8)))
        return a


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# bdm_alloc_fn / bdm_free_fn of include/bdm.h
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class TorchAllocator:
    """bdm_create_ex callbacks backed by torch's CUDA caching allocator, so the library's
    per-agent, grid and exchange buffers come out of (and return to) the pool the
    caller's tensors live in.  Keeps the counts a test can check."""

    def __init__(self, device: int):
        import torch
        self.device = int(device)
        self.live = {}
        self.n_alloc = self.n_free = 0
        self.bytes_live = self.bytes_peak = 0

        def _alloc(nbytes, stream, _user):
            try:
                st = stream if stream else torch.cuda.current_stream(self.device).cuda_stream
                p = torch.cuda.caching_allocator_alloc(int(nbytes), self.device, st)
            except Exception:  # out of memory: the library reports BDM_ECAPACITY
                return None
            self.live[p] = int(nbytes)
            self.n_alloc += 1
            self.bytes_live += int(nbytes)
            self.bytes_peak = max(self.bytes_peak, self.bytes_live)
            return p

        def _free(p, _stream, _user):
            nb = self.live.pop(p, None)
            if nb is None:
                return
            self.n_free += 1
            self.bytes_live -= nb
            torch.cuda.caching_allocator_delete(p)

        self.alloc_cb, self.free_cb = ALLOC_FN(_alloc), FREE_FN(_free)


class Engine:
    """Owns a bdm_handle (library workspace on one device).  With `allocator` (e.g. a
    TorchAllocator) the workspace is taken from the caller's pool (bdm_create_ex)."""

    def __init__(self, device: int = 0, max_agents: int = 1, max_ghosts: int = 0, allocator=None):
        self.lib = load_library()
        h = ctypes.c_void_p()
        self.allocator = allocator  # keeps the callbacks alive as long as the handle
        if allocator is None and max_ghosts == 0:
            _check(self.lib.bdm_create(ctypes.byref(h), int(device), int(max_agents)))
        else:
            _check(self.lib.bdm_create_ex(
                ctypes.byref(h), int(device), int(max_agents), int(max_ghosts),
                allocator.alloc_cb if allocator else ALLOC_FN(0),
                allocator.free_cb if allocator else FREE_FN(0), None))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.bdm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- calls of bdm.h
    def init_spheres(self, agents: Agents, n, seed=1, side=160.0, d_lo=10.0, d_width=0.0,
                     d_random=False, id0=0, stream=None):
        ca = agents.c()
        _check(self.lib.bdm_init_spheres(self.h, ctypes.byref(ca), int(id0), int(n), int(seed),
                                         float(side), float(d_lo), float(d_width),
                                         int(bool(d_random)), _stream_ptr(stream)))
        agents.n = int(n)

    def grid_build(self, agents: Agents, radius: float = 0.0, stream=None, ghosts=None):
        ca = agents.c()
        cg = ghosts.c() if ghosts is not None else None
        _check(self.lib.bdm_grid_build(self.h, ctypes.byref(ca),
                                       ctypes.byref(cg) if cg is not None else None,
                                       float(radius), _stream_ptr(stream)))

    # -------------------------------------------------------------- x-slab device side
    def local_frame(self, agents: Agents, out, stream=None):
        """bdm_local_frame into the device tensor `out` (4 float64)."""
        ca = agents.c()
        _check(self.lib.bdm_local_frame(self.h, ctypes.byref(ca), _ptr(out), _stream_ptr(stream)))

    def set_frame(self, frame):
        """bdm_set_frame (device tensor of 4 float64, kept alive by the caller) or None."""
        self._frame_ref = frame
        _check(self.lib.bdm_set_frame(self.h, _ptr(frame) if frame is not None else None))

    def pack_slab(self, agents: Agents, lo: float, hi: float, margin: float, what: int,
                  to_left: Agents, to_right: Agents, stream=None):
        """bdm_pack_slab; synchronizes; sets to_left.n, to_right.n (and agents.n for a
        migration); returns (n_left, n_right)."""
        import torch
        if not hasattr(self, "_pack_counts"):
            self._pack_counts = torch.zeros(3, dtype=torch.int64, pin_memory=True)
        ca, cl, cr = agents.c(), to_left.c(), to_right.c()
        _check(self.lib.bdm_pack_slab(self.h, ctypes.byref(ca), float(lo), float(hi),
                                      float(margin), int(what), ctypes.byref(cl),
                                      ctypes.byref(cr), ctypes.c_void_p(self._pack_counts.data_ptr()),
                                      _stream_ptr(stream)))
        self.sync(stream)
        nl, nr, rem = (int(v) for v in self._pack_counts)
        to_left.n, to_right.n = nl, nr
        if what == PACK_MIGRATE:
            agents.n = rem
        return nl, nr

    # ---- x-slab exchange behind the C ABI (bdm_dist_init / bdm_aura_exchange)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load_library().bdm_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return buf.raw

    def dist_init(self, uid: bytes, rank: int, nranks: int, lo: float, hi: float,
                  radius: float = 0.0):
        """Join the NCCL x-slab group (collective over the ranks)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(self.lib.bdm_dist_init(self.h, ctypes.cast(buf, ctypes.c_void_p), int(rank),
                                      int(nranks), float(lo), float(hi), float(radius)))

    def aura_exchange(self, local: Agents, ghosts: Agents, stream=None):
        """Frame + migration + aura for this step (one host synchronization).  Grows
        `local` / `ghosts` when the arrivals do not fit and completes the exchange."""
        cl, cg = local.c(), ghosts.c()
        st = self.lib.bdm_aura_exchange(self.h, ctypes.byref(cl), ctypes.byref(cg),
                                        _stream_ptr(stream))
        local.n, ghosts.n = cl.n, cg.n
        if st == BDM_ECAPACITY:
            self._finish_pending(local, ghosts, stream)
        else:
            _check(st)

    def _finish_pending(self, local: Agents, ghosts: Agents, stream=None):
        need = (ctypes.c_int64 * 2)()
        _check(self.lib.bdm_aura_pending(self.h, ctypes.cast(need, ctypes.c_void_p)))
        if need[0] > local.capacity:
            local.grow(int(need[0] * 5 // 4 + 1024))
        if need[1] > ghosts.capacity:
            ghosts.grow(int(need[1] * 5 // 4 + 1024))
        cl, cg = local.c(), ghosts.c()
        _check(self.lib.bdm_aura_finish(self.h, ctypes.byref(cl), ctypes.byref(cg),
                                        _stream_ptr(stream)))
        local.n, ghosts.n = cl.n, cg.n

    @staticmethod
    def dist_init_virtual(engines, lo, hi, radius: float = 0.0):
        """G contexts of this process (one device) as G virtual x-slabs."""
        G = len(engines)
        hs = (ctypes.c_void_p * G)(*[e.h for e in engines])
        los = (ctypes.c_double * G)(*[float(v) for v in lo])
        his = (ctypes.c_double * G)(*[float(v) for v in hi])
        _check(load_library().bdm_dist_init_virtual(ctypes.cast(hs, ctypes.c_void_p), G,
                                                     ctypes.cast(los, ctypes.c_void_p),
                                                     ctypes.cast(his, ctypes.c_void_p),
                                                     float(radius)))

    @staticmethod
    def aura_exchange_virtual(engines, locals_, ghosts, stream=None):
        G = len(engines)
        hs = (ctypes.c_void_p * G)(*[e.h for e in engines])
        cl = (CAgents * G)(*[a.c() for a in locals_])
        cg = (CAgents * G)(*[g.c() for g in ghosts])
        st = load_library().bdm_aura_exchange_virtual(ctypes.cast(hs, ctypes.c_void_p), G,
                                                      ctypes.cast(cl, ctypes.c_void_p),
                                                      ctypes.cast(cg, ctypes.c_void_p),
                                                      _stream_ptr(stream))
        for k in range(G):
            locals_[k].n, ghosts[k].n = cl[k].n, cg[k].n
        if st == BDM_ECAPACITY:
            for k in range(G):
                engines[k]._finish_pending(locals_[k], ghosts[k], stream)
        else:
            _check(st)

    def append(self, dst: Agents, src: Agents, stream=None):
        cd, cs = dst.c(), src.c()
        _check(self.lib.bdm_append(self.h, ctypes.byref(cd), ctypes.byref(cs), _stream_ptr(stream)))
        dst.n = int(cd.n)

    def mech_step(self, agents: Agents, params: Params, stream=None):
        """bdm_mech_step over the grid of the preceding grid_build (locals only are
        written)."""
        ca = agents.c()
        cp = params.c()
        _check(self.lib.bdm_mech_step(self.h, ctypes.byref(ca), ctypes.byref(cp),
                                      _stream_ptr(stream)))

    def step(self, agents: Agents, params: Params, stream=None, sync: bool = False,
             retries: int = 3):
        """grid build + mechanics step, asynchronous on `stream` by default (errors and
        a grid-slot overflow surface at the next bdm_sync).  With sync=True, checks the
        latched device conditions and, on a grid-slot overflow, grows the slot array and
        re-issues the step (the caller's arrays are untouched by an overflowed step)."""
        for _ in range(retries + 1):
            if params.boundary == 2:  # toroidal: bdm_step builds the grid on the torus (R52)
                ca, cp = agents.c(), params.c()
                _check(self.lib.bdm_step(self.h, ctypes.byref(ca), ctypes.byref(cp),
                                         _stream_ptr(stream)))
            else:
                self.grid_build(agents, params.radius, stream)
                self.mech_step(agents, params, stream)
            if not sync:
                return
            st = self.lib.bdm_sync(self.h, _stream_ptr(stream))
            if st == BDM_ECAPACITY:
                gi = self.grid_info()
                _check(self.lib.bdm_reserve(self.h, 0, int(gi["nslots"] * 3 // 2)))
                continue
            _check(st)
            return
        raise BdmError(BDM_ECAPACITY, "grid slot capacity could not be satisfied")

    def grow_divide(self, agents: Agents, params: Params, growth: float, v_max: float,
                    stream=None) -> int:
        """bdm_grow_divide; synchronizes, updates agents.n and returns it.  Raises
        BdmError(BDM_ECAPACITY) if the arrays cannot hold the daughters."""
        import torch
        if not hasattr(self, "_n_out"):
            self._n_out = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        ca = agents.c()
        cp = params.c()
        _check(self.lib.bdm_grow_divide(self.h, ctypes.byref(ca), ctypes.byref(cp), float(growth),
                                        float(v_max), ctypes.c_void_p(self._n_out.data_ptr()),
                                        _stream_ptr(stream)))
        self.sync(stream)
        agents.n = int(self._n_out[0])
        return agents.n

    def sir_step(self, agents: Agents, params: Params, side: float, radius: float,
                 p_inf: float, p_rec: float, stream=None, sync: bool = True):
        """bdm_sir_step.  With sync=True returns the counts (S, I, R, new infections); if
        the infected index was too small (the step is then a no-op) it is enlarged to n
        and the step re-issued."""
        import torch
        if not hasattr(self, "_sir_counts"):
            self._sir_counts = torch.zeros(4, dtype=torch.int64, pin_memory=True)
        for attempt in range(2):
            ca = agents.c()
            cp = params.c()
            _check(self.lib.bdm_sir_step(self.h, ctypes.byref(ca), ctypes.byref(cp), float(side),
                                         float(radius), float(p_inf), float(p_rec),
                                         ctypes.c_void_p(self._sir_counts.data_ptr()),
                                         _stream_ptr(stream)))
            if not sync:
                return None
            st = self.lib.bdm_sync(self.h, _stream_ptr(stream))
            if st == BDM_ECAPACITY and attempt == 0 and getattr(self, "_sir_autogrow", True):
                self.set_option("sir_index_capacity", max(int(agents.n), 1))
                continue
            _check(st)
            return [int(v) for v in self._sir_counts]
        return None

    # ---------------------------------------------------------------- row f4
    def diffuse(self, u_in, u_out, grid: CGrid3, nu: float, mu: float, dt: float, stream=None):
        """bdm_diffuse: one Eq. 4.3 step from the (nz, ny, nx) float64 tensor u_in to
        u_out (distinct)."""
        _check(self.lib.bdm_diffuse(self.h, _ptr(u_in), _ptr(u_out), ctypes.byref(grid),
                                    float(nu), float(mu), float(dt), _stream_ptr(stream)))

    def secrete(self, agents: Agents, type_, type_sel: int, q: float, u, grid: CGrid3,
                stream=None):
        """bdm_secrete: agents of type type_sel add q to the cell of their position."""
        ca = agents.c()
        _check(self.lib.bdm_secrete(self.h, ctypes.byref(ca), _ptr(type_), int(type_sel),
                                    float(q), _ptr(u), ctypes.byref(grid), _stream_ptr(stream)))

    def chemotaxis(self, agents: Agents, type_, type_sel: int, weight: float, u, grid: CGrid3,
                   stream=None):
        """bdm_chemotaxis: agents of type type_sel move by weight x the normalized
        gradient of u at their cell."""
        ca = agents.c()
        _check(self.lib.bdm_chemotaxis(self.h, ctypes.byref(ca), _ptr(type_), int(type_sel),
                                       float(weight), _ptr(u), ctypes.byref(grid),
                                       _stream_ptr(stream)))

    def soma_step(self, agents: Agents, type_, grids, spares, grid: CGrid3, nu: float,
                  mu: float, dt: float, q: float, weight: float, stream=None):
        """One soma-clustering step (reading R39): secretion of every type
        into its own substance, chemotaxis of every type, one diffusion step of every
        substance from grids[t] into spares[t].  Returns (grids, spares) swapped: the new
        concentrations and the buffers free for the next step."""
        for t, u in enumerate(grids):
            self.secrete(agents, type_, t, q, u, grid, stream)
        for t, u in enumerate(grids):
            self.chemotaxis(agents, type_, t, weight, u, grid, stream)
        for u, v in zip(grids, spares):
            self.diffuse(u, v, grid, nu, mu, dt, stream)
        return list(spares), list(grids)

    def onco_step(self, agents: Agents, age, p: "COncoParams", id_next: int, stream=None):
        """bdm_onco_step (Alg. 4 + removal, row f2); age is an int32/uint32 device tensor
        indexed by id.  Synchronizes, sets agents.n and returns the new id_next.  Raises
        BdmError(BDM_ECAPACITY) with nothing modified if the population would exceed the
        capacity of agents or of age."""
        import torch
        if not hasattr(self, "_onco_out"):
            self._onco_out = torch.zeros(2, dtype=torch.int64, pin_memory=True)
        ca = agents.c()
        _check(self.lib.bdm_onco_step(self.h, ctypes.byref(ca), _ptr(age), int(age.numel()),
                                      ctypes.byref(p),
                                      int(id_next), ctypes.c_void_p(self._onco_out.data_ptr()),
                                      _stream_ptr(stream)))
        st = self.lib.bdm_sync(self.h, _stream_ptr(stream))
        if st != BDM_OK:
            _check(st)
        n, nxt = (int(v) for v in self._onco_out)
        agents.n = n
        return nxt

    # ---- row f3: delta + LZ4 aura codec (bdm_aura_*)
    def aura_reference(self, msg: Agents, ref: Agents, stream=None):
        """ref := msg in ascending id order (the reference both sides keep, R46)."""
        cm, cr = msg.c(), ref.c()
        _check(self.lib.bdm_aura_reference(self.h, ctypes.byref(cm), ctypes.byref(cr),
                                           _stream_ptr(stream)))
        ref.n = cr.n

    def aura_encode(self, msg: Agents, ref: Agents, out, stream=None) -> int:
        """Stream of msg against ref into the uint8 device tensor out; returns its bytes."""
        cm, cr = msg.c(), ref.c()
        size = ctypes.c_int64()
        _check(self.lib.bdm_aura_encode(self.h, ctypes.byref(cm), ctypes.byref(cr), _ptr(out),
                                        int(out.numel()), ctypes.byref(size), _stream_ptr(stream)))
        return int(size.value)

    def aura_decode(self, stream_buf, nbytes: int, ref: Agents, msg: Agents, stream=None):
        """msg := the message of stream_buf[:nbytes] decoded against ref (sets msg.n)."""
        cr, cm = ref.c(), msg.c()
        _check(self.lib.bdm_aura_decode(self.h, _ptr(stream_buf), int(nbytes), ctypes.byref(cr),
                                        ctypes.byref(cm), _stream_ptr(stream)))
        msg.n = cm.n

    def aura_max_size(self, nref: int, n: int) -> int:
        return int(self.lib.bdm_aura_max_size(int(nref), int(n)))

    def cfg3_step(self, agents: Agents, params: Params, growth: float, v_max: float,
                  stream=None) -> int:
        """One proliferation step (R15): grid + mechanics on the snapshot, then
        growth/division at the post-mechanics positions."""
        self.step(agents, params, stream=stream, sync=True)
        return self.grow_divide(agents, params, growth, v_max, stream=stream)

    def step_host(self, host_in: Agents, host_out: Agents, dev: Agents, params: Params,
                  stream=None):
        ci, co, cd, cp = host_in.c(), host_out.c(), dev.c(), params.c()
        _check(self.lib.bdm_step_host(self.h, ctypes.byref(ci), ctypes.byref(co),
                                      ctypes.byref(cd), ctypes.byref(cp), _stream_ptr(stream)))
        host_out.n = host_in.n
        dev.n = host_in.n

    def run_host(self, host: Agents, dev: Agents, params: Params, steps: int, chunks: int = 8,
                 stream=None):
        """`steps` end-to-end steps on the pinned host state `host` (in place), uploads
        of step k+1 overlapping downloads of step k chunk by chunk (bdm_run_host)."""
        ch, cd, cp = host.c(), dev.c(), params.c()
        _check(self.lib.bdm_run_host(self.h, ctypes.byref(ch), ctypes.byref(cd), ctypes.byref(cp),
                                     int(steps), int(chunks), _stream_ptr(stream)))
        dev.n = host.n

    def sync(self, stream=None):
        _check(self.lib.bdm_sync(self.h, _stream_ptr(stream)))

    def try_sync(self, stream=None) -> int:
        return int(self.lib.bdm_sync(self.h, _stream_ptr(stream)))

    def reserve(self, max_agents: int = 0, nslots: int = 0):
        _check(self.lib.bdm_reserve(self.h, int(max_agents), int(nslots)))

    def stats(self) -> dict:
        s = CStats()
        _check(self.lib.bdm_get_stats(self.h, ctypes.byref(s)))
        return {k: getattr(s, k) for k in ("cand", "nbr", "cont", "n_static", "n_moved",
                                           "launches")}

    def grid_info(self) -> dict:
        g = CGridInfo()
        _check(self.lib.bdm_get_grid_info(self.h, ctypes.byref(g)))
        return {"R": g.R, "L": g.L, "origin": list(g.origin), "upper": list(g.upper),
                "dims": list(g.dims), "nslots": g.nslots, "slot_capacity": g.slot_capacity}

    def neighbor_pairs(self, agents: Agents, radius: float = 0.0, stream=None):
        """Sorted numpy uint64 array of (id_i << 32 | id_j) through the GPU grid."""
        import numpy as np
        import torch
        ca = agents.c()
        cnt = ctypes.c_int64()
        cap = 1
        buf = torch.empty(cap, dtype=torch.int64, device=agents.x.device)
        st = self.lib.bdm_neighbor_pairs(self.h, ctypes.byref(ca), float(radius), _ptr(buf), cap,
                                         ctypes.byref(cnt), _stream_ptr(stream))
        if st == BDM_ECAPACITY and cnt.value > cap:
            cap = cnt.value
            buf = torch.empty(cap, dtype=torch.int64, device=agents.x.device)
            ca = agents.c()
            st = self.lib.bdm_neighbor_pairs(self.h, ctypes.byref(ca), float(radius), _ptr(buf),
                                             cap, ctypes.byref(cnt), _stream_ptr(stream))
        _check(st)
        return np.sort(buf[:cnt.value].cpu().numpy().view(np.uint64))

    def set_option(self, name: str, value: int):
        _check(self.lib.bdm_set_option(self.h, name.encode(), int(value)))

    def peak_dfma(self):
        v = ctypes.c_double()
        n = ctypes.c_int32()
        _check(self.lib.bdm_peak_dfma(self.h, ctypes.byref(v), ctypes.byref(n)))
        return v.value, n.value

    def selftest_recip_div(self, n: int, seed: int = 1) -> int:
        """Mismatches of the SIR step's shared-reciprocal quotients against IEEE
        division on n random operands (bdm_selftest_recip_div)."""
        v = ctypes.c_ulonglong()
        _check(self.lib.bdm_selftest_recip_div(self.h, int(n), int(seed), ctypes.byref(v)))
        return int(v.value)
