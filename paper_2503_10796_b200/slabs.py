"""x-slab decomposition across GPUs (TeraAgent).

Space is cut into mutually exclusive x-slabs [lo_g, hi_g), one per GPU, the outer
slabs unbounded ("partitioning grid").  Every iteration:

  1. migration  agents that left their slab move to the neighbour that owns their new
                position (|displacement| <= 3 um << slab width, so only
                adjacent slabs are involved and the collective lookup of P:6124-6126
                never triggers);
  2. frame      element-wise MIN all-reduce of (min x, min y, min z, -max d): every
                rank builds its grid on the same global lattice, so the canonical
                summation order (R9) -- and therefore every bit of the result -- is the
                same as on one GPU (R12, R24);
  3. aura       agents within R(1+2^-20) of a slab border are copied to the neighbour
                (rebuilt every iteration); optionally as a
                delta-encoded + LZ4 stream against a reference both sides keep and
                refresh every `ref_every` iterations (row f3, P:6291-6356,
                bdm_aura_*), for links slower than NVLink;
  4. compute    bdm_grid_build(locals, ghosts) + bdm_mech_step (locals only).

The device side (packing, appending, frames, the step) is libbdm.so; the transport is
pluggable: ``DistTransport`` uses torch.distributed point-to-point (NCCL over NVLink on
GPUs; gloo for the CPU tests), ``LocalTransport`` connects several slabs living in one
process (the "virtual slab" mode used to test the GPU path on one device).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .bdm import PACK_AURA, PACK_MIGRATE, Agents, Engine, Params

F64_FIELDS = ("x", "y", "z", "diameter")
I32_FIELDS = ("id", "flags")
GHOST_MARGIN = 1.0 + 2.0**-20   # R24: aura margin R(1+2^-20) = the box edge L (R5)


def slab_bounds(g: int, G: int, side: float):
    """[lo, hi) of slab g of G over [0, side) in x; the outer slabs are unbounded."""
    lo = -math.inf if g == 0 else g * side / G
    hi = math.inf if g == G - 1 else (g + 1) * side / G
    return lo, hi


# ---------------------------------------------------------------------------- device ops
class LibOps:
    """Device side of one slab, backed by a libbdm context (one GPU).  With DistTransport
    the stream must be torch's current stream: the transport's NCCL calls and payload
    copies are ordered on it, and the library's packing and appending must be too."""

    def __init__(self, engine: Engine, device="cuda", stream=None):
        self.eng = engine
        self.device = device
        self.stream = stream
        self._frame = None

    def buffer(self, capacity: int, like: Agents = None) -> Agents:
        vol = like is not None and like.volume is not None
        return Agents.empty(max(int(capacity), 1), device=self.device, volume=vol)

    def pack(self, agents: Agents, lo, hi, margin, what):
        cap = max(agents.n, 1)
        left, right = self.buffer(cap, agents), self.buffer(cap, agents)
        self.eng.pack_slab(agents, lo, hi, margin, what, left, right, stream=self.stream)
        return left, right

    def append(self, dst: Agents, src: Agents):
        if src is not None and src.n > 0:
            self.eng.append(dst, src, stream=self.stream)

    def local_frame(self, agents: Agents):
        import torch
        out = torch.empty(4, dtype=torch.float64, device=self.device)
        self.eng.local_frame(agents, out, stream=self.stream)
        return out

    def set_frame(self, frame):
        self._frame = frame
        self.eng.set_frame(frame)

    def compute(self, agents: Agents, ghosts: Agents, params: Params):
        for _ in range(4):
            self.eng.grid_build(agents, params.radius, stream=self.stream, ghosts=ghosts)
            self.eng.mech_step(agents, params, stream=self.stream)
            st = self.eng.try_sync(self.stream)
            if st == -2:  # grid slots exceeded: the step was a no-op, grow and re-issue
                gi = self.eng.grid_info()
                self.eng.reserve(0, int(gi["nslots"] * 3 // 2))
                continue
            if st != 0:
                self.eng.sync(self.stream)
            return
        raise RuntimeError("grid capacity could not be satisfied")

    # row f3: aura codec (device byte streams)
    def empty_ref(self) -> Agents:
        a = self.buffer(1)
        a.n = 0
        return a

    def aura_reference(self, msg: Agents) -> Agents:
        ref = self.buffer(max(msg.n, 1))
        self.eng.aura_reference(msg, ref, stream=self.stream)
        return ref

    def aura_encode(self, msg: Agents, ref: Agents):
        import torch
        buf = torch.empty(self.eng.aura_max_size(ref.n, msg.n), dtype=torch.uint8,
                          device=self.device)
        nb = self.eng.aura_encode(msg, ref, buf, stream=self.stream)
        return buf[:nb]

    def aura_decode(self, stream_bytes, ref: Agents) -> Agents:
        hdr = stream_bytes[:40].cpu().numpy().tobytes() if stream_bytes.numel() >= 40 else b""
        nnew = int.from_bytes(hdr[16:24], "little") if hdr else 0
        out = self.buffer(max(ref.n + nnew, 1))
        self.eng.aura_decode(stream_bytes, int(stream_bytes.numel()), ref, out, stream=self.stream)
        return out

    # payload <-> tensors (views, no copy)
    def to_payload(self, a: Agents):
        fields = {k: getattr(a, k)[:a.n] for k in F64_FIELDS + I32_FIELDS}
        if a.volume is not None:
            fields["volume"] = a.volume[:a.n]
        return fields

    def from_payload(self, fields, n: int) -> Agents:
        a = self.buffer(max(n, 1), None)
        if "volume" in fields:
            import torch
            a.volume = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)
        for k, t in fields.items():
            getattr(a, k)[:n].copy_(t[:n])
        a.n = n
        return a

    def payload_template(self, n: int, with_volume: bool):
        import torch
        f = {k: torch.empty(max(n, 1), dtype=torch.float64, device=self.device) for k in F64_FIELDS}
        f.update({k: torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
                  for k in I32_FIELDS})
        if with_volume:
            f["volume"] = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)
        return f


# ---------------------------------------------------------------------------- transports
class LocalTransport:
    """Slabs of one process (virtual-slab mode): slab g's left buffer goes to g-1."""

    def exchange(self, sends: dict) -> dict:
        recv = {}
        for g in sends:
            from_left = sends[g - 1][1] if (g - 1) in sends else None
            from_right = sends[g + 1][0] if (g + 1) in sends else None
            recv[g] = (from_left, from_right)
        return recv

    def exchange_bytes(self, sends: dict) -> dict:
        return self.exchange(sends)

    def allreduce_min(self, frames: dict) -> dict:
        import torch
        vals = list(frames.values())
        m = vals[0].clone()
        for v in vals[1:]:
            m = torch.minimum(m, v.to(m.device))
        return {g: m.to(v.device) for g, v in frames.items()}


class DistTransport:
    """One slab per process (slab id = rank); torch.distributed point-to-point with the
    left and right neighbours (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU)."""

    def __init__(self, ops, device, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.ops = ops
        self.device = device
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _p2p(self, ops_list):
        if ops_list:
            for req in self.dist.batch_isend_irecv(ops_list):
                req.wait()

    def exchange(self, sends: dict) -> dict:
        import torch
        dist = self.dist
        (g, (to_left, to_right)), = sends.items()
        left, right = g - 1, g + 1
        has_l, has_r = left >= 0, right < self.world
        with_vol = to_left is not None and getattr(to_left, "volume", None) is not None
        # 1) counts
        cnt_out = torch.tensor([to_left.n if to_left is not None else 0,
                                to_right.n if to_right is not None else 0],
                               dtype=torch.int64, device=self.device)
        cnt_in = torch.zeros(2, dtype=torch.int64, device=self.device)  # from left, from right
        ops = []
        if has_l:
            ops += [dist.P2POp(dist.isend, cnt_out[0:1], left, self.group),
                    dist.P2POp(dist.irecv, cnt_in[0:1], left, self.group)]
        if has_r:
            ops += [dist.P2POp(dist.isend, cnt_out[1:2], right, self.group),
                    dist.P2POp(dist.irecv, cnt_in[1:2], right, self.group)]
        self._p2p(ops)
        n_from_l, n_from_r = (int(v) for v in cnt_in.cpu())
        # 2) payloads, field by field (fixed order)
        recv_l = self.ops.payload_template(n_from_l, with_vol) if has_l else None
        recv_r = self.ops.payload_template(n_from_r, with_vol) if has_r else None
        send_l = self.ops.to_payload(to_left) if (has_l and to_left is not None) else None
        send_r = self.ops.to_payload(to_right) if (has_r and to_right is not None) else None
        ops = []
        for k in sorted((send_l or send_r or recv_l or recv_r or {}).keys()):
            if has_l and to_left.n > 0:
                ops.append(dist.P2POp(dist.isend, send_l[k].contiguous(), left, self.group))
            if has_l and n_from_l > 0:
                ops.append(dist.P2POp(dist.irecv, recv_l[k][:n_from_l], left, self.group))
            if has_r and to_right.n > 0:
                ops.append(dist.P2POp(dist.isend, send_r[k].contiguous(), right, self.group))
            if has_r and n_from_r > 0:
                ops.append(dist.P2POp(dist.irecv, recv_r[k][:n_from_r], right, self.group))
        self._p2p(ops)
        from_l = self.ops.from_payload(recv_l, n_from_l) if has_l else None
        from_r = self.ops.from_payload(recv_r, n_from_r) if has_r else None
        return {g: (from_l, from_r)}

    def exchange_bytes(self, sends: dict) -> dict:
        """Byte streams (uint8 tensors) with the two neighbours: sizes, then bytes."""
        import torch
        dist = self.dist
        (g, (to_left, to_right)), = sends.items()
        left, right = g - 1, g + 1
        has_l, has_r = left >= 0, right < self.world
        size = lambda t: int(t.numel()) if t is not None else 0  # noqa: E731
        cnt_out = torch.tensor([size(to_left), size(to_right)], dtype=torch.int64,
                               device=self.device)
        cnt_in = torch.zeros(2, dtype=torch.int64, device=self.device)
        ops = []
        if has_l:
            ops += [dist.P2POp(dist.isend, cnt_out[0:1], left, self.group),
                    dist.P2POp(dist.irecv, cnt_in[0:1], left, self.group)]
        if has_r:
            ops += [dist.P2POp(dist.isend, cnt_out[1:2], right, self.group),
                    dist.P2POp(dist.irecv, cnt_in[1:2], right, self.group)]
        self._p2p(ops)
        n_l, n_r = (int(v) for v in cnt_in.cpu())
        recv_l = torch.empty(max(n_l, 1), dtype=torch.uint8, device=self.device)
        recv_r = torch.empty(max(n_r, 1), dtype=torch.uint8, device=self.device)
        ops = []
        if has_l and size(to_left) > 0:
            ops.append(dist.P2POp(dist.isend, to_left.contiguous(), left, self.group))
        if has_l and n_l > 0:
            ops.append(dist.P2POp(dist.irecv, recv_l[:n_l], left, self.group))
        if has_r and size(to_right) > 0:
            ops.append(dist.P2POp(dist.isend, to_right.contiguous(), right, self.group))
        if has_r and n_r > 0:
            ops.append(dist.P2POp(dist.irecv, recv_r[:n_r], right, self.group))
        self._p2p(ops)
        return {g: (recv_l[:n_l] if has_l else None, recv_r[:n_r] if has_r else None)}

    def allreduce_min(self, frames: dict) -> dict:
        (g, f), = frames.items()
        t = f.clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return {g: t}


# ---------------------------------------------------------------------------- protocol
@dataclass
class Slab:
    g: int
    lo: float
    hi: float
    ops: object
    agents: object
    ghosts: object = None


class SlabDomain:
    """The per-iteration protocol over the slabs this process owns (one per process with
    DistTransport, several with LocalTransport)."""

    def __init__(self, slabs: list, transport, params: Params, aura_codec: bool = False,
                 ref_every: int = 10):
        self.slabs = {s.g: s for s in slabs}
        self.tr = transport
        self.params = params
        self.last = {}
        self.aura_codec = aura_codec
        self.ref_every = max(int(ref_every), 1)
        self.iteration = 0
        # row f3 references: (slab, "L"/"R") -> the last message sent that way, and
        # (slab, "L"/"R") -> the receiver's copy of what arrives from that side
        self.ref_send, self.ref_recv = {}, {}

    def migrate(self):
        sends = {g: s.ops.pack(s.agents, s.lo, s.hi, 0.0, PACK_MIGRATE) for g, s in self.slabs.items()}
        recvs = self.tr.exchange(sends)
        moved = 0
        for g, s in self.slabs.items():
            fl, fr = recvs[g]
            for part in (fl, fr):
                if part is not None and part.n > 0:
                    s.ops.append(s.agents, part)
                    moved += part.n
        return moved

    def frame(self):
        frames = {g: s.ops.local_frame(s.agents) for g, s in self.slabs.items()}
        glob = self.tr.allreduce_min(frames)
        for g, s in self.slabs.items():
            s.ops.set_frame(glob[g])
        f = next(iter(glob.values()))
        return [float(v) for v in (f.cpu() if hasattr(f, "cpu") else f)]

    def aura(self, R: float):
        margin = R * GHOST_MARGIN
        sends = {g: s.ops.pack(s.agents, s.lo, s.hi, margin, PACK_AURA) for g, s in self.slabs.items()}
        self.aura_bytes = [0, 0]  # (stream bytes, raw 40 B/agent bytes) sent
        if self.aura_codec:
            recvs = self._aura_codec(sends)
        else:
            recvs = self.tr.exchange(sends)
        n_ghosts = 0
        for g, s in self.slabs.items():
            fl, fr = recvs[g]
            parts = [p for p in (fl, fr) if p is not None and p.n > 0]
            total = sum(p.n for p in parts)
            ghosts = s.ops.buffer(max(total, 1), None)
            ghosts.n = 0
            for p in parts:
                s.ops.append(ghosts, p)
            s.ghosts = ghosts if total > 0 else None
            n_ghosts += total
        return n_ghosts

    def _aura_codec(self, sends: dict) -> dict:
        """Row f3: each direction encodes against the reference both ends hold; every
        ref_every iterations both ends replace it with the message just exchanged (the
        receiver's decoded copy has the same agents, so the id-ordered references stay
        identical).  Ghost order does not enter a result (R9)."""
        refresh = self.iteration % self.ref_every == 0
        streams = {}
        for g, (left, right) in sends.items():
            ops = self.slabs[g].ops
            enc = []
            for side, msg in (("L", left), ("R", right)):
                ref = self.ref_send.get((g, side))
                if ref is None:
                    ref = ops.empty_ref()
                st = ops.aura_encode(msg, ref)
                self.aura_bytes[0] += int(st.numel())
                self.aura_bytes[1] += 40 * msg.n
                enc.append(st)
                if refresh:
                    self.ref_send[(g, side)] = ops.aura_reference(msg)
            streams[g] = tuple(enc)
        got = self.tr.exchange_bytes(streams)
        recvs = {}
        for g, (bl, br) in got.items():
            ops = self.slabs[g].ops
            parts = []
            for side, st in (("L", bl), ("R", br)):  # from the left / right neighbour
                if st is None:
                    parts.append(None)
                    continue
                ref = self.ref_recv.get((g, side))
                if ref is None:
                    ref = ops.empty_ref()
                msg = ops.aura_decode(st, ref)
                if refresh:
                    self.ref_recv[(g, side)] = ops.aura_reference(msg)
                parts.append(msg)
            recvs[g] = tuple(parts)
        return recvs

    def step(self):
        moved = self.migrate()
        f = self.frame()
        R = self.params.radius if self.params.radius > 0 else -f[3]
        ng = self.aura(R)
        for g, s in self.slabs.items():
            s.ops.compute(s.agents, s.ghosts, self.params)
        self.last = {"migrated": moved, "ghosts": ng, "frame": f}
        if self.aura_codec:
            self.last["aura_stream_bytes"], self.last["aura_raw_bytes"] = self.aura_bytes
        self.iteration += 1
        return self.last


# ---------------------------------------------------------------------------- native path
class NativeSlabDomain:
    """The x-slab step through the C ABI: one bdm_aura_exchange per slab and step (the
    global frame, migration and aura in one call with one host synchronization, over
    NCCL between ranks, or bdm_aura_exchange_virtual for several slabs of this process
    on one device), then bdm_grid_build(local, ghosts) + bdm_mech_step, with no further
    host synchronization.  The protocol is the one-round variant of SlabDomain: every
    rank packs its leavers and its aura from the same pre-step state, and keeps its own
    leavers as ghosts (they now belong to the neighbour and sit at the shared border),
    so migration and aura travel together.

    engines[k] / agents[k]: the slabs of this process (k = its rank in the group).  With
    uid (bytes from Engine.nccl_unique_id on rank 0, broadcast by the caller) the single
    slab joins the NCCL group `rank` of `nranks`; without it the slabs form a virtual
    group."""

    def __init__(self, engines, agents, bounds, params: Params, stream=None, uid=None,
                 rank: int = 0, nranks: int = 1, ghost_capacity: int = 1 << 16):
        self.engines = list(engines)
        self.agents = list(agents)
        self.params = params
        self.stream = stream
        self.virtual = uid is None
        vol = self.agents[0].volume is not None
        self.ghosts = [Agents.empty(ghost_capacity, device=a.x.device, volume=vol) for a in self.agents]
        if self.virtual:
            Engine.dist_init_virtual(self.engines, [b[0] for b in bounds], [b[1] for b in bounds],
                                     params.radius)
        else:
            assert len(self.engines) == 1
            lo, hi = bounds[0]
            self.engines[0].dist_init(uid, rank, nranks, lo, hi, params.radius)
        self.last = {}

    def exchange(self):
        if self.virtual:
            Engine.aura_exchange_virtual(self.engines, self.agents, self.ghosts, stream=self.stream)
        else:
            self.engines[0].aura_exchange(self.agents[0], self.ghosts[0], stream=self.stream)

    def step(self):
        self.exchange()
        for e, a, g in zip(self.engines, self.agents, self.ghosts):
            e.grid_build(a, self.params.radius, stream=self.stream, ghosts=g if g.n > 0 else None)
            e.mech_step(a, self.params, stream=self.stream)
        self.last = {"ghosts": sum(g.n for g in self.ghosts), "local": sum(a.n for a in self.agents)}
        return self.last

    def check(self):
        """Synchronize and report any latched device condition (grid slots, ...)."""
        for e in self.engines:
            e.sync(self.stream)
