"""Test double for the device side of the x-slab protocol (paper_2503_10796_b200/slabs.py).

Implements LibOps' interface on the CPU with numpy and the oracle, so that the protocol
(migration, global frame, aura, transports) can be exercised in world_size-2 gloo runs
without a GPU.  Test infrastructure only; the product path uses LibOps (libbdm.so).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

F64 = ("x", "y", "z", "diameter")
I32 = ("id", "flags")


class NpAgents:
    def __init__(self, n=0, arrays=None):
        self.arrays = arrays if arrays is not None else {
            "x": np.zeros(n), "y": np.zeros(n), "z": np.zeros(n), "diameter": np.zeros(n),
            "id": np.zeros(n, np.uint32), "flags": np.zeros(n, np.uint32)}
        self.n = n
        self.volume = None

    @staticmethod
    def from_state(s, mask=None):
        idx = np.arange(len(s["x"])) if mask is None else np.nonzero(mask)[0]
        arr = {"x": s["x"][idx].copy(), "y": s["y"][idx].copy(), "z": s["z"][idx].copy(),
               "diameter": s["d"][idx].copy(), "id": s["id"][idx].astype(np.uint32),
               "flags": s["flags"][idx].astype(np.uint32)}
        return NpAgents(len(idx), arr)

    def state(self):
        a = self.arrays
        return {"x": a["x"][:self.n], "y": a["y"][:self.n], "z": a["z"][:self.n],
                "d": a["diameter"][:self.n], "id": a["id"][:self.n], "flags": a["flags"][:self.n]}

    def take(self, idx):
        return NpAgents(len(idx), {k: v[:self.n][idx].copy() for k, v in self.arrays.items()})


class OracleOps:
    def __init__(self, params):
        self.params = params          # oracle MechParams template (without frame)
        self.frame = None

    def buffer(self, capacity, like=None):
        a = NpAgents(0)
        return a

    def pack(self, agents, lo, hi, margin, what):
        x = agents.arrays["x"][:agents.n]
        if what == 1:   # migrate
            left, right = x < lo, x >= hi
        else:
            left, right = x < lo + margin, x >= hi - margin
        L, R = agents.take(np.nonzero(left)[0]), agents.take(np.nonzero(right)[0])
        if what == 1:
            keep = agents.take(np.nonzero(~(left | right))[0])
            agents.arrays, agents.n = keep.arrays, keep.n
        return L, R

    def append(self, dst, src):
        if src is None or src.n == 0:
            return
        for k in dst.arrays:
            dst.arrays[k] = np.concatenate([dst.arrays[k][:dst.n], src.arrays[k][:src.n]])
        dst.n += src.n

    def local_frame(self, agents):
        a = agents.arrays
        n = agents.n
        if n == 0:
            return torch.full((4,), float("inf"), dtype=torch.float64)
        return torch.tensor([a["x"][:n].min(), a["y"][:n].min(), a["z"][:n].min(),
                             -a["diameter"][:n].max()], dtype=torch.float64)

    def set_frame(self, frame):
        self.frame = [float(v) for v in frame]

    def compute(self, agents, ghosts, params):
        both = NpAgents(0, {k: v[:agents.n].copy() for k, v in agents.arrays.items()})
        both.n = agents.n
        if ghosts is not None:
            self.append(both, ghosts)
        f = self.frame
        p = oracle.mech_params(k=self.params.k, gamma=self.params.gamma, dt=self.params.dt,
                               max_disp=self.params.max_disp,
                               force_threshold=self.params.force_threshold,
                               detect_static=bool(self.params.detect_static),
                               frame=(f[0], f[1], f[2], -f[3]))
        out, _ = oracle.mech_step(both.state(), p, sample=np.arange(agents.n))
        agents.arrays["x"][:agents.n] = out["x"]
        agents.arrays["y"][:agents.n] = out["y"]
        agents.arrays["z"][:agents.n] = out["z"]
        agents.arrays["flags"][:agents.n] = out["flags"]

    # row f3 codec (byte streams as torch uint8 CPU tensors)
    def empty_ref(self):
        return NpAgents(0)

    def aura_reference(self, msg):
        return NpAgents.from_state(oracle.aura_reference(msg.state()))

    def aura_encode(self, msg, ref):
        st = oracle.aura_encode(msg.state(), ref.state())
        return torch.frombuffer(bytearray(st), dtype=torch.uint8)

    def aura_decode(self, stream_bytes, ref):
        return NpAgents.from_state(oracle.aura_decode(stream_bytes.numpy().tobytes(), ref.state()))

    # payloads for DistTransport (torch CPU tensors)
    def to_payload(self, a):
        p = {k: torch.from_numpy(np.ascontiguousarray(a.arrays[k][:a.n], np.float64)) for k in F64}
        p.update({k: torch.from_numpy(np.ascontiguousarray(a.arrays[k][:a.n], np.uint32).view(np.int32))
                  for k in I32})
        return p

    def payload_template(self, n, with_volume):
        p = {k: torch.empty(max(n, 1), dtype=torch.float64) for k in F64}
        p.update({k: torch.empty(max(n, 1), dtype=torch.int32) for k in I32})
        return p

    def from_payload(self, fields, n):
        arr = {k: fields[k][:n].numpy().copy() for k in F64}
        arr.update({k: fields[k][:n].numpy().view(np.uint32).copy() for k in I32})
        return NpAgents(n, arr)
