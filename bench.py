#!/usr/bin/env python
"""bench.py -- agent-updates/s of the B200 mechanics step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg1|cfg5] [--no-e2e] [--no-cpu-baseline]

One "step" = one pass of the whole hot path over the agents: grid build (a1-a4:
reduce, keys, histogram, scan, scatter, in-box id order, gather) + mechanics (a5-a9:
static test, 27-box scan, Eq. 4.1 force, canonical sum, capped displacement) -- all in
libbdm.so kernels behind the C ABI.  The workload at N=1 is configs[1] (cfg2: 10M
agents, d ~ U[8,12] um, 50 % volume fraction, static skip on).  Inputs (440 MB of
SoA) exceed the 126 MB L2, so no flush is needed between steps; the state evolves
from step to step exactly as the simulation does.

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (oracle/, the
from-scratch reference of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "agent-updates/sec per mechanics step (fp64) and % of HBM/fp64 roofline"
UNIT = "agent-updates/s"

# Algorithmic work per agent-update: bytes the method must move
# and fp64 pipe instructions the method must issue.
B_ALG_PER_AGENT = 72.0           # x,y,z,d read (32) + x,y,z write (24) + key/perm (16)
B_ALG_STATIC_EXTRA = 8.0         # flags read + write with detect_static
# the mechanics kernel alone: sorted x,y,z,d + id + flags read (40), x,y,z,d + id + flags
# written to the caller's arrays (40)
MECH_ALG_BYTES_PER_AGENT = 80.0
FP64_PER_CAND, FP64_PER_NBR, FP64_PER_CONT, FP64_PER_AGENT = 7.0, 3.0, 60.0, 40.0


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.dev = device_index
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - NVML missing
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ CPU oracle legs
_ORC = {}  # state read by the forked oracle workers (shared copy-on-write)


def host_cpu():
    """(cpu model, cores available to this process, logical cpus)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return model, cores, os.cpu_count()


def _mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return 16.0


def _orc_mech_slice(bounds):
    import numpy as np
    import oracle
    lo, hi, _ = bounds
    oracle.mech_step(_ORC["s"], _ORC["p"], sample=np.arange(lo, hi, dtype=np.int64))
    return hi - lo


def _orc_sir_slice(bounds):
    import numpy as np
    import oracle
    lo, hi, t = bounds
    c = _ORC["cfg"]
    oracle.sir_step_sample(_ORC["s"], c.side, c.radius, c.p_inf, c.p_rec, c.seed, t,
                           np.arange(lo, hi, dtype=np.int64))
    return hi - lo


class OracleAllCores:
    """The oracle (oracle/, single-threaded C, unchanged) on all host cores.  One worker
    process per core (fork), each running the oracle's step in its sample mode on a
    disjoint contiguous slice of the agents, all on the same full start-of-step state;
    every worker builds the step's grid index itself, as the oracle's step does.  The
    per-agent results are the oracle's, so the slices together are one whole step."""

    def __init__(self, state, params=None, kind="mech", sir_cfg=None, bytes_per_agent=24.0):
        import multiprocessing as mp

        import numpy as np
        _ORC.clear()
        _ORC.update(s=state, p=params, cfg=sir_cfg)
        self.kind = kind
        self.n = len(state["x"])
        self.model, cores, self.ncpu = host_cpu()
        per_worker_gb = bytes_per_agent * 1.5 * self.n / 2**30 + 0.2
        self.workers = max(1, min(cores, int(0.6 * _mem_available_gb() / per_worker_gb)))
        edges = np.linspace(0, self.n, self.workers + 1).astype(np.int64)
        self.bounds = [(int(edges[k]), int(edges[k + 1])) for k in range(self.workers)
                       if edges[k + 1] > edges[k]]
        self.pool = mp.get_context("fork").Pool(self.workers)

    def step(self, t=0):
        fn = _orc_mech_slice if self.kind == "mech" else _orc_sir_slice
        t0 = time.perf_counter()
        done = sum(self.pool.map(fn, [(lo, hi, t) for lo, hi in self.bounds], chunksize=1))
        dt = time.perf_counter() - t0
        assert done == self.n
        return dt

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self):
        return {"cores": self.workers, "threads": self.workers, "nproc": self.ncpu,
                "cpu_model": self.model}


def _mech_state(cfg):
    """A mid-run state of a mechanics config: the seeded population with every agent
    flagged MOVED (at tau = 0 nearly every agent moves each step, so no agent is a
    static candidate, as in the GPU's timed steps)."""
    import oracle
    s = oracle.init_spheres(cfg.n, cfg.seed, cfg.side, cfg.d_lo, cfg.d_width, cfg.d_random)
    s["flags"][:] = 1
    return s


def cpu_baseline_mech(cfg, steps=1, note=""):
    """The oracle on all host cores, `steps` whole steps of `cfg` (rank 0, N = 1)."""
    import oracle
    oracle.build()
    s = _mech_state(cfg)
    p = oracle.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                           force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    orc = OracleAllCores(s, p)
    try:
        times = [orc.step() for _ in range(steps)]
    finally:
        orc.close()
    t = statistics.median(times)
    return {"value": cfg.n / t, "unit": UNIT, "kind": "oracle", **orc.describe(),
            "sample": f"{steps} whole oracle step(s) of {cfg.name} ({cfg.n} agents, mid-run "
                      f"flags), agents split over {orc.workers} worker processes (the oracle's "
                      f"sample mode, disjoint slices; each worker builds the step's grid index); "
                      f"median {t:.2f} s{note}"}


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle (as it stands) on all host cores (rank 0 only),
    on cfg2, the metric's workload.  Each step is one whole oracle step of a cube of the
    cfg2 population (same density, diameter mix, static skip) whose size is chosen so the
    --steps K --warmup W run ends in about --ref-budget seconds (150 by default)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    steps, warm = args.steps, min(args.warmup, 3)
    cal_n = 500_000
    cal = W.cfg2_scaled(cal_n)
    orc = OracleAllCores(_mech_state(cal), oracle.mech_params(detect_static=True))
    try:
        t_cal = orc.step()
    finally:
        orc.close()
    per_agent = t_cal / cal_n
    n = int(min(W.CFG2.n, max(200_000, args.ref_budget / ((steps + warm) * per_agent))))
    cfg = W.cfg2_scaled(n) if n < W.CFG2.n else W.CFG2
    orc = OracleAllCores(_mech_state(cfg), oracle.mech_params(detect_static=True))
    try:
        for _ in range(warm):
            orc.step()
        times = [orc.step() for _ in range(steps)]
    finally:
        orc.close()
    dt = sum(times)
    value = cfg.n * steps / dt
    sample = (f"each step = one whole oracle mechanics step of a {cfg.n}-agent cube of the cfg2 "
              f"population (same density, diameter mix, static skip; mid-run flags), the "
              f"agents split over {orc.workers} worker processes (oracle sample mode)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg2 (configs[1]), spatial sample", "agents_per_step": cfg.n,
                   "full_workload_agents": W.CFG2.n},
        "step_ms": {"median": statistics.median(times) * 1e3,
                    "p90": sorted(times)[int(0.9 * (len(times) - 1))] * 1e3},
        "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", **orc.describe(),
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args, ws, rank, local):
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params

    if ws > 1 or args.force_slabs:
        return run_slabs(args, ws, rank, local)
    if args.config == "cfg3":
        return run_cfg3(args, ws, rank, local)
    if args.config == "cfg4":
        return run_cfg4(args, ws, rank, local)
    if args.config == "soma":
        return run_soma(args, ws, rank, local)
    if args.config == "onco":
        return run_onco(args, ws, rank, local)
    if args.config == "aura":
        return run_aura(args, ws, rank, local)
    torch.cuda.set_device(local)
    cfg = W.PRESETS[args.config]
    eng = Engine(local, cfg.n)
    eng.set_option("mech_kernel", args.mech_kernel)
    eng.set_option("fuse_reduce", 1)   # a1 of the next step fused into the mechanics epilogue
    eng.set_option("tile_order", args.tile_order)
    eng.set_option("tile_depth", args.tile_depth)
    a = Agents.empty(cfg.n)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo,
                         d_width=cfg.d_width, d_random=cfg.d_random, stream=stream)
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    # first step sizes the grid; reserve slot headroom (+8 tiles/axis) for the growth of
    # the open-boundary space over the run so no timed step overflows
    eng.step(a, params, stream=stream, sync=True)
    gi = eng.grid_info()
    T = [(d + 3) // 4 + 8 for d in gi["dims"]]
    if args.tile_order:
        T = [(t + 7) // 8 * 8 for t in T]
    eng.reserve(0, T[0] * T[1] * T[2] * 64)
    if args.shuffle:  # row f1: a random memory order (the sorted order is undone)
        torch.cuda.synchronize()
        g = torch.Generator(device="cuda")
        g.manual_seed(11)
        p = torch.randperm(cfg.n, device="cuda", generator=g)
        for f in ("x", "y", "z", "diameter", "id", "flags"):
            t = getattr(a, f)
            t[:cfg.n] = t[:cfg.n][p]
        torch.cuda.synchronize()
    eng.set_option("sort_every", args.sort_every)
    for _ in range(max(args.warmup - 1, 0)):
        eng.step(a, params, stream=stream)
    # work counters of a representative step (the last warm-up step)
    pst = Params(**{**params.__dict__, "collect_stats": True})
    eng.step(a, pst, stream=stream)
    st_before = eng.stats()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.stats()["launches"]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for k in range(K):
            e0, e1, e2 = ev[k]
            e0.record(stream)
            eng.grid_build(a, params.radius, stream=stream)
            e1.record(stream)
            eng.mech_step(a, params, stream=stream)
            e2.record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = eng.stats()["launches"] - launches0
    rc = eng.try_sync(stream)
    if rc != 0:
        raise SystemExit(f"a timed step failed (bdm status {rc}); rerun")
    total_ms = start.elapsed_time(stop)
    grid_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(K)]
    mech_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(K)]
    step_ms = [ev[k][0].elapsed_time(ev[k][2]) for k in range(K)]
    eng.step(a, pst, stream=stream)
    st_after = eng.stats()
    clocks = clk.summary()
    graph = _graph_steps(eng, a, params, stream, K) if not args.no_graph else None

    ms_step = total_ms / K
    value = cfg.n / (ms_step * 1e-3)

    # roofline of the dominant kernel (k_mech): fp64-pipe bound
    avg = lambda k: 0.5 * (st_before[k] + st_after[k])  # noqa: E731
    cand, nbr, cont, nstat = avg("cand"), avg("nbr"), avg("cont"), avg("n_static")
    fp64_per_launch = (FP64_PER_CAND * cand + FP64_PER_NBR * nbr + FP64_PER_CONT * cont +
                       FP64_PER_AGENT * cfg.n)
    mech_avg_s = statistics.mean(mech_ms) * 1e-3
    peaks, peak_src = _peaks()
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = clocks["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    fp64_peak = sm_count * 64 * max_mhz * 1e6  # fp64 lane-instructions/s at max clock
    achieved = fp64_per_launch / mech_avg_s
    b_alg = (B_ALG_PER_AGENT + (B_ALG_STATIC_EXTRA if cfg.detect_static else 0.0)) * cfg.n
    hbm_peak = peaks["hbm_gbs"] * 1e9
    t_roof = max(b_alg / hbm_peak, fp64_per_launch / fp64_peak)
    dfma_meas, _ = eng.peak_dfma()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": {"cfg2": "cfg2 (configs[1])", "cfg5": "cfg5 (configs[4]) on one GPU"}
                   .get(cfg.name, cfg.name),
                   "agents": cfg.n, "side_um": cfg.side, "diameter": "U[8,12] um"
                   if cfg.d_random else f"{cfg.d_lo} um", "detect_static": cfg.detect_static,
                   "dt": cfg.dt, "max_displacement_um": cfg.max_disp,
                   "l2": "inputs (44 B/agent SoA) larger than L2; no flush",
                   "parallelism": f"{ws} GPU"},
        **({"f1": {"tile_order": args.tile_order, "sort_every": args.sort_every,
                   "shuffled_start": args.shuffle}}
           if (args.tile_order, args.sort_every, args.shuffle) != (0, 1, False) else {}),
        "roofline": {"bound": "alu", "kernel": "k_mech (a5-a9)",
                     "achieved": achieved / 1e12, "peak": fp64_peak / 1e12,
                     "unit": "T fp64-inst/s", "frac": achieved / fp64_peak,
                     **_traffic_keys(_traffic("k_mech_tile6" if cfg.name == "cfg2" else "k_mech_tile6_cfg5",
                                              MECH_ALG_BYTES_PER_AGENT * cfg.n)
                                     if cfg.name in ("cfg2", "cfg5") else None),
                     "peak_source": f"{sm_count} SMs x 64 fp64 lanes x {max_mhz:.0f} MHz "
                                    f"(guide unit counts, max clock); measured DFMA "
                                    f"{dfma_meas / 1e12:.2f} T/s",
                     "work_per_launch": {"cand": cand, "nbr": nbr, "cont": cont,
                                         "static": nstat, "fp64_inst": fp64_per_launch},
                     "mech_ms": statistics.mean(mech_ms), "grid_ms": statistics.mean(grid_ms)},
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms_step * 1e-3),
                          "hbm_term_ms": b_alg / hbm_peak * 1e3,
                          "fp64_term_ms": fp64_per_launch / fp64_peak * 1e3,
                          "hbm_peak_gbs": peaks["hbm_gbs"], "hbm_peak_source": peak_src},
        "step_ms": _dist(step_ms),
        "graph": graph,
        "clocks": clocks,
        "gpu_launches": launches,
    }

    if cfg.name == "cfg5":
        # 1.7e9 agents: a pinned host copy in and out (2 x 68 GB) plus a second device SoA
        # do not fit beside the 178 GB the step itself holds
        line["e2e"] = None
        line["e2e_note"] = "not measured for cfg5: host/device staging copies do not fit"
    elif not args.no_e2e:
        line["e2e"] = measure_e2e(eng, cfg, params, stream)
    if not args.no_cpu_baseline and rank == 0 and ws == 1:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if cfg.name == "cfg2" and args.strong_steps > 0:
        # T_1 of the strong-scaled cfg5 (1.7B agents on this one GPU), for S_N = T_1 / T_N
        eng.close()
        del a, eng
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        try:
            line["strong_cfg5"] = _slab_phase(args, 1, 0, local, True, args.strong_steps, 2)
        except Exception as e:  # noqa: BLE001 (reported in the line)
            line["strong_cfg5"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    print(json.dumps(line), flush=True)


def _graph_steps(eng, a, params, stream, K):
    """The same step (grid build + mechanics, a fixed launch sequence at fixed n) captured
    once as a CUDA graph and replayed K times: the device time per step without the
    host's launch path.  (The JSON line's value is the direct-launch number.)"""
    import torch
    try:
        eng.step(a, params, stream=stream)          # leaves the fused extent for the graph
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            g.capture_begin(capture_error_mode="relaxed")
            eng.grid_build(a, params.radius, stream=stream)
            eng.mech_step(a, params, stream=stream)
            g.capture_end()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):  # replays go to the current stream
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(K):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        rc = eng.try_sync(stream)
        if rc != 0:
            return {"error": f"bdm status {rc} after the graph replays"}
        return {"ms_per_step": e0.elapsed_time(e1) / K, "replays": K,
                "kernels_per_step": "grid build + mechanics, one graph"}
    except Exception as e:  # noqa: BLE001 (reported in the line)
        return {"error": f"{type(e).__name__}: {e}"[:200]}


def _dist(ms):
    """Per-step device times (CUDA events): mean, median, p90, min, max (ms)."""
    v = sorted(ms)
    return {"mean": statistics.mean(v), "median": statistics.median(v),
            "p90": v[min(len(v) - 1, int(math.ceil(0.9 * len(v))) - 1)], "min": v[0], "max": v[-1],
            "n": len(v)}


def _common(metric_value, ms_step, ws, args, config, clocks, launches, dtype="f64"):
    return {"metric": METRIC, "value": metric_value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic", "config": config, "clocks": clocks, "gpu_launches": launches}


def run_cfg3(args, ws, rank, local):
    """configs[2]: proliferation 1M -> 256M agents over 20 steps (every step has a
    different N; the value is the aggregate sum(N_t) / sum(t_step))."""
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    torch.cuda.set_device(local)
    cfg = W.CFG3
    steps = min(args.steps, cfg.steps)
    cap = cfg.n * 2 ** ((steps + 1) // 2 + 1)
    cap = min(cap, 300_000_000)
    eng = Engine(local, cfg.n)
    a = Agents.empty(cap, volume=True)
    stream = torch.cuda.Stream()
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, stream=stream)
    a.volume[:cfg.n].copy_((torch.pi / 6.0) * (a.diameter[:cfg.n] ** 3))
    torch.cuda.synchronize()
    params = Params(seed=cfg.seed, dt=cfg.dt, max_displacement=cfg.max_disp)
    # workspace for the final population and for the finest grid (R = 8 um), reserved
    # before timing so no step pays for an allocation
    tiles = int(math.ceil((cfg.side + 2 * steps * cfg.max_disp) / cfg.d_lo / 4.0)) + 8
    eng.reserve(cap, tiles ** 3 * 64)
    per_step = []
    launches0 = eng.stats()["launches"]
    with ClockSampler(local) as clk:
        for t in range(steps):
            params.step = t
            n0 = a.n
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            eng.step(a, params, stream=stream, sync=True)
            eng.grow_divide(a, params, W.CFG3_GROWTH, W.CFG3_V_MAX, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            per_step.append((n0, e0.elapsed_time(e1)))
    total_agents = sum(n for n, _ in per_step)
    total_ms = sum(ms for _, ms in per_step)
    launches = eng.stats()["launches"] - launches0
    clocks = clk.summary()
    # the same 20 steps again (deterministic: the same populations) with the work counters
    # on, untimed, for each step's roofline; and the oracle on the host cores on the
    # populations of the steps it finishes in seconds (N <= 4M)
    peaks, src = _peaks()
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = clocks["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    fp64_peak = sm_count * 64 * max_mhz * 1e6
    hbm_peak = peaks["hbm_gbs"] * 1e9
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, stream=stream)
    a.volume[:cfg.n].copy_((torch.pi / 6.0) * (a.diameter[:cfg.n] ** 3))
    torch.cuda.synchronize()
    pst = Params(seed=cfg.seed, dt=cfg.dt, max_displacement=cfg.max_disp, collect_stats=True)
    rows, orc_rows = [], []
    do_orc = not args.no_cpu_baseline and rank == 0
    for t, (n_t, ms) in enumerate(per_step):
        pst.step = t
        if do_orc and a.n <= 4_000_000:
            h = a.numpy()
            orc_rows.append((a.n, _oracle_mech_time({k: h[k] for k in ("x", "y", "z", "d", "id", "flags")},
                                                    cfg)))
        eng.step(a, pst, stream=stream, sync=True)
        st = eng.stats()
        eng.grow_divide(a, pst, W.CFG3_GROWTH, W.CFG3_V_MAX, stream=stream)
        fp64 = (FP64_PER_CAND * st["cand"] + FP64_PER_NBR * st["nbr"] + FP64_PER_CONT * st["cont"] +
                FP64_PER_AGENT * n_t)
        b_alg = (B_ALG_PER_AGENT + 16.0) * n_t    # + volume read and write (cfg3)
        t_roof = max(b_alg / hbm_peak, fp64 / fp64_peak)
        rows.append({"n": n_t, "ms": round(ms, 4), "t_roof_ms": round(t_roof * 1e3, 4),
                     "frac": round(t_roof * 1e3 / ms, 4), "cand_per_agent": st["cand"] / n_t,
                     "cont_per_agent": st["cont"] / n_t,
                     "bound": "fp64" if fp64 / fp64_peak > b_alg / hbm_peak else "hbm"})
    t_roof_total = sum(r["t_roof_ms"] for r in rows)
    line = _common(total_agents / (total_ms * 1e-3), total_ms / steps, ws, args,
                   {"workload": "cfg3 (configs[2])", "initial_agents": cfg.n,
                    "final_agents": a.n, "steps": steps, "per_step": rows,
                    "l2": "inputs larger than L2 from step 1 (48 B/agent x >= 1M)"},
                   clocks, launches)
    line["roofline"] = {"bound": "alu", "kernel": "whole step (grid + mechanics + division), per step",
                        "t_roof_total_ms": t_roof_total, "t_total_ms": total_ms,
                        "frac": t_roof_total / total_ms,
                        "peak_source": f"fp64: {sm_count} SMs x 64 lanes x {max_mhz:.0f} MHz; "
                                       f"HBM {peaks['hbm_gbs']} GB/s ({src})",
                        "work": "fp64 term 7 cand + 3 nbr + 60 cont + 40 per agent; 88 B/agent"}
    if orc_rows:
        on = sum(n for n, _ in orc_rows)
        ot = sum(t for _, (t, _) in orc_rows)
        line["cpu_baseline"] = {"value": on / ot, "unit": UNIT, "kind": "oracle", **orc_rows[0][1][1],
                                "sample": f"the oracle on all host cores, one whole step on each of "
                                          f"the populations of steps 0-{len(orc_rows) - 1} "
                                          f"(N = {orc_rows[0][0]} .. {orc_rows[-1][0]}; taken from the "
                                          f"GPU run, which is bit-identical to the oracle's); the "
                                          f"later, denser steps (up to {a.n} agents) are not run"}
    line["note"] = "proliferation: per-step rate and roofline in config.per_step; dense late steps run the dense-box kernel"
    print(json.dumps(line), flush=True)


def _oracle_mech_time(state, cfg):
    """One whole oracle mechanics step of `state` on all host cores -> (s, describe)."""
    import oracle
    oracle.build()
    p = oracle.mech_params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_disp=cfg.max_disp,
                           force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    orc = OracleAllCores(state, p)
    try:
        dt = orc.step()
    finally:
        orc.close()
    return dt, orc.describe()


def run_cfg4(args, ws, rank, local):
    """configs[3]: SIR on 100M point agents, HBM-bound (x, y, z, state read + written)."""
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    torch.cuda.set_device(local)
    cfg = W.CFG4
    eng = Engine(local, 1)
    a = Agents.empty(cfg.n, state=True)
    stream = torch.cuda.Stream()
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=0.0, stream=stream)
    torch.cuda.synchronize()
    a.state[:cfg.n_infected] = 1
    a.id = None       # ids == index: the Philox counter uses the index (no id traffic)
    a.diameter = None
    a.flags = None
    torch.cuda.synchronize()
    params = Params(seed=cfg.seed)
    for t in range(args.warmup):
        params.step = t
        eng.sir_step(a, params, cfg.side, cfg.radius, cfg.p_inf, cfg.p_rec, stream=stream)
    K = args.steps
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    launches0 = eng.stats()["launches"]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        evs[0].record(stream)
        for k in range(K):
            params.step = args.warmup + k
            eng.sir_step(a, params, cfg.side, cfg.radius, cfg.p_inf, cfg.p_rec, stream=stream,
                         sync=False)
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
    rc = eng.try_sync(stream)
    if rc != 0:
        raise SystemExit(f"a timed SIR step failed (bdm status {rc})")
    counts = [int(v) for v in eng._sir_counts]
    ms = evs[0].elapsed_time(evs[K]) / K
    peaks, src = _peaks()
    b_alg = 50.0 * cfg.n    # x, y, z read + write (48 B) + state read + write (2 B)
    ach = b_alg / (ms * 1e-3)
    line = _common(cfg.n / (ms * 1e-3), ms, ws, args,
                   {"workload": "cfg4 (configs[3])", "agents": cfg.n, "side_m": cfg.side,
                    "radius_m": cfg.radius, "p_inf": cfg.p_inf, "p_rec": cfg.p_rec,
                    "l2": "inputs (2.5 GB) larger than L2; no flush",
                    "counts_after": {"S": counts[0], "I": counts[1], "R": counts[2]}},
                   clk.summary(), eng.stats()["launches"] - launches0)
    line["roofline"] = {"bound": "hbm", "kernel": "k_sir_update + k_sir_collect (whole step)",
                        "achieved": ach / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": ach / (peaks["hbm_gbs"] * 1e9),
                        **_traffic_keys(_traffic("k_sir_update", b_alg)),
                        "peak_source": src, "alg_bytes_per_agent": 50}
    line["step_ms"] = _dist([evs[k].elapsed_time(evs[k + 1]) for k in range(K)])
    if not args.no_cpu_baseline and rank == 0:
        line["cpu_baseline"] = cpu_baseline_sir(a, cfg)
    print(json.dumps(line), flush=True)


def cpu_baseline_sir(a, cfg, steps=3):
    """The SIR oracle on all host cores, `steps` whole steps of the cfg4 population (the
    GPU's current state copied to the host; each worker process updates a disjoint slice
    of the agents with orc_sir_step_sample, which builds the infected index itself)."""
    import numpy as np
    import oracle
    oracle.build()
    n = a.n
    s = {"x": a.x[:n].cpu().numpy(), "y": a.y[:n].cpu().numpy(), "z": a.z[:n].cpu().numpy(),
         "state": a.state[:n].cpu().numpy(), "id": np.arange(n, dtype=np.uint32)}
    orc = OracleAllCores(s, kind="sir", sir_cfg=cfg, bytes_per_agent=8.0)
    try:
        times = [orc.step(t) for t in range(steps)]
    finally:
        orc.close()
    t = statistics.median(times)
    return {"value": n / t, "unit": UNIT, "kind": "oracle", **orc.describe(),
            "sample": f"{steps} whole oracle SIR steps of the cfg4 population ({n} agents), "
                      f"agents split over {orc.workers} worker processes; median {t:.2f} s"}


def _traffic(kernel, alg_bytes):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/r02/traffic.json, written from the .ncu-rep summaries), next to the
    algorithmic bytes of the same launch; None if there is no capture."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    return {"dram_bytes_per_launch": t["dram_bytes_per_launch"],
            **{k: t[k] for k in ("issue_active_pct", "fp64_pipe_active_pct", "warp_inst_per_launch",
                                 "warp_inst_per_agent", "fp64_thread_inst_per_agent",
                                 "shared_wavefronts_per_launch", "shared_bank_conflict_wavefronts_per_launch",
                                 "warps_active_pct") if k in t},
            "alg_bytes_per_launch": alg_bytes,
            "ratio": t["dram_bytes_per_launch"] / alg_bytes if alg_bytes else None,
            "source": t["source"], "capture_workload": t["workload"]}


def _traffic_keys(t):
    """roofline.traffic = DRAM bytes per launch (the number the contract names), with
    the capture it comes from and the algorithmic bytes beside it."""
    return {"traffic": t["dram_bytes_per_launch"] if t else None, "traffic_detail": t}


def run_soma(args, ws, rank, local):
    """soma clustering steps (secretion, chemotaxis, Eq. 4.3 diffusion
    of two substances on res^3 fp64 grids).  The stencil kernel is HBM-bound: 8 B read +
    8 B written per grid point and step."""
    import torch
    from paper_2503_10796_b200 import Agents, CGrid3, Engine
    torch.cuda.set_device(local)
    cfg = W.SOMA
    eng = Engine(local, cfg.n)
    a = Agents.empty(cfg.n)
    stream = torch.cuda.Stream()
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d, stream=stream)
    ttype = (torch.arange(cfg.n, device="cuda") % 2).to(torch.uint8)
    r = cfg.res
    dx = cfg.side / r
    grid = CGrid3.make(r, r, r, (0.0, 0.0, 0.0), dx)
    grids = [torch.zeros((r, r, r), dtype=torch.float64, device="cuda") for _ in range(2)]
    spares = [torch.zeros_like(grids[0]) for _ in range(2)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            grids, spares = eng.soma_step(a, ttype, grids, spares, grid, cfg.nu, cfg.mu, cfg.dt,
                                          cfg.q, cfg.weight, stream=stream)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    launches0 = eng.stats()["launches"]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(K):
            e0, e1, e2 = ev[k]
            e0.record(stream)
            for t, u in enumerate(grids):
                eng.secrete(a, ttype, t, cfg.q, u, grid, stream)
            for t, u in enumerate(grids):
                eng.chemotaxis(a, ttype, t, cfg.weight, u, grid, stream)
            e1.record(stream)
            for u, v in zip(grids, spares):
                eng.diffuse(u, v, grid, cfg.nu, cfg.mu, cfg.dt, stream)
            e2.record(stream)
            grids, spares = spares, grids
        torch.cuda.synchronize()
    ms = [ev[k][0].elapsed_time(ev[k][2]) for k in range(K)]
    dms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(K)]
    ms_step = statistics.mean(ms)
    points = 2 * r ** 3
    peaks, src = _peaks()
    d_s = statistics.mean(dms) * 1e-3 / 2          # one substance's k_diffuse launch
    ach = 16.0 * r ** 3 / d_s
    line = {
        "metric": "grid-point updates/s (Eq. 4.3 diffusion, soma clustering; SURVEY 8(f) f4)",
        "value": points / (ms_step * 1e-3), "unit": "point-updates/s", "n_gpus": ws,
        "steps": K, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "soma clustering (SURVEY 8(f) row f4)", **cfg.to_dict(),
                   "substances": 2, "grid_points": points,
                   "agent_updates_per_s": cfg.n / (ms_step * 1e-3),
                   "l2": "grids (1 GiB each) larger than L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "k_diffuse (one substance, one step)",
                     "achieved": ach / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": ach / (peaks["hbm_gbs"] * 1e9),
                     **_traffic_keys(_traffic("k_diffuse_tma", 16.0 * r ** 3)),
                     "peak_source": src, "alg_bytes_per_point": 16,
                     "diffuse_ms": statistics.mean(dms) / 2},
        "clocks": clk.summary(), "gpu_launches": eng.stats()["launches"] - launches0,
    }
    print(json.dumps(line), flush=True)


def run_onco(args, ws, rank, local):
    """tumor-spheroid steps (grid + mechanics, then Alg. 4 with
    removal and division).  Every step has a different N; value = sum(N_t) / sum(t)."""
    import torch
    from paper_2503_10796_b200 import Agents, COncoParams, Engine, Params
    torch.cuda.set_device(local)
    cfg = W.ONCO
    steps = min(args.steps, cfg.steps)
    cap = int(cfg.n * 1.6) + 1024
    eng = Engine(local, cap)
    a = Agents.empty(cap, volume=True)
    stream = torch.cuda.Stream()
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                     d_random=True, stream=stream)
    torch.cuda.synchronize()
    d = a.diameter[:cfg.n]
    a.volume[:cfg.n].copy_((math.pi / 6.0) * (d * d * d))
    # ages (R44): floor(u32(Philox(seed, (id, 0xFFFFFFFC, 2)).w0) * 120), drawn on the host
    # by the same counter-based generator the init uses (ids 0..n-1)
    age = torch.zeros(2 * cap, dtype=torch.int32, device="cuda")
    age[:cfg.n].copy_(_onco_ages(cfg.n, cfg.seed, cfg.max_age0))
    mp = Params(k=2.0, gamma=1.0, dt=1.0, max_displacement=1.0, force_threshold=1.8)
    tiles = int(math.ceil((cfg.side + 2 * steps) / 10.0 / 4.0)) + 8
    eng.reserve(cap, tiles ** 3 * 64)
    id_next = cfg.n
    if args.warmup:  # one untimed step on a scratch copy: lazy buffers, first launches
        w = Agents.empty(cap, volume=True)
        for f in ("x", "y", "z", "diameter", "id", "flags", "volume"):
            getattr(w, f)[:a.n].copy_(getattr(a, f)[:a.n])
        w.n = a.n
        eng.step(w, mp, stream=stream)
        eng.onco_step(w, age.clone(), COncoParams.make(step=0, seed=cfg.seed), id_next,
                      stream=stream)
        torch.cuda.synchronize()
        del w
    per_step = []
    launches0 = eng.stats()["launches"]
    with ClockSampler(local) as clk:
        for t in range(steps):
            n0 = a.n
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            eng.step(a, mp, stream=stream)
            e1.record(stream)
            id_next = eng.onco_step(a, age, COncoParams.make(step=t, seed=cfg.seed), id_next,
                                    stream=stream)
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(stream)
            torch.cuda.synchronize()
            per_step.append((n0, e0.elapsed_time(e2), e0.elapsed_time(e1)))
    total_agents = sum(n for n, _, _ in per_step)
    total_ms = sum(ms for _, ms, _ in per_step)
    line = _common(total_agents / (total_ms * 1e-3), total_ms / steps, ws, args,
                   {"workload": "tumor spheroid cells (SURVEY 8(f) row f2)", **asdict_safe(cfg),
                    "final_agents": a.n, "id_next": id_next,
                    "per_step": [{"n": n, "ms": round(ms, 4), "mech_ms": round(m, 4)}
                                 for n, ms, m in per_step],
                    "l2": "inputs larger than L2 (>= 48 B/agent x 1M); no flush"},
                   clk.summary(), eng.stats()["launches"] - launches0)
    line["roofline"] = None
    line["note"] = "the step is the cfg2-type mechanics + the behaviour/removal pass (HBM-bound)"
    print(json.dumps(line), flush=True)


def run_aura(args, ws, rank, local):
    """the aura a cfg2 x-slab sends its neighbour (agents within the
    interaction radius of the slab plane x = side/2), encoded against a reference taken
    at the first timed step (delta + LZ4, bdm_aura_encode) and decoded back, once per
    mechanics step.  value = aura agents encoded per second; the sizes compare the
    stream with the raw 40 B/agent message and with LZ4 alone (empty reference)."""
    import torch
    from paper_2503_10796_b200 import Agents, Engine, Params
    torch.cuda.set_device(local)
    cfg = W.CFG2
    eng = Engine(local, cfg.n)
    eng.set_option("fuse_reduce", 1)
    a = Agents.empty(cfg.n)
    stream = torch.cuda.Stream()
    eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                     d_random=cfg.d_random, stream=stream)
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    force_threshold=cfg.force_threshold, detect_static=cfg.detect_static)
    for _ in range(args.warmup):
        eng.step(a, params, stream=stream)
    torch.cuda.synchronize()
    mid, margin = 0.5 * cfg.side, cfg.d_lo + cfg.d_width      # R = max diameter
    fields = (("x", "x"), ("y", "y"), ("z", "z"), ("diameter", "diameter"), ("id", "id"),
              ("flags", "flags"))

    def aura():
        sel = torch.nonzero((a.x[:a.n] - mid).abs() < margin).squeeze(1)
        m = Agents.empty(int(sel.numel()) + 1)
        for f, _ in fields:
            getattr(m, f)[:sel.numel()].copy_(getattr(a, f)[:a.n][sel])
        m.n = int(sel.numel())
        return m

    msg0 = aura()
    ref = Agents.empty(msg0.n + 1)
    eng.aura_reference(msg0, ref, stream=stream)
    empty = Agents.empty(1)
    empty.n = 0
    # warm-up of the codec (workspace allocation, kernel attributes)
    wbuf = torch.empty(eng.aura_max_size(ref.n, msg0.n), dtype=torch.uint8, device="cuda")
    wout = Agents.empty(2 * msg0.n + 1)
    eng.aura_decode(wbuf, eng.aura_encode(msg0, ref, wbuf, stream=stream), ref, wout, stream=stream)
    rows = []
    launches0 = eng.stats()["launches"]
    with ClockSampler(local) as clk:
        for t in range(args.steps):
            eng.step(a, params, stream=stream)
            torch.cuda.synchronize()
            m = aura()
            cap = eng.aura_max_size(ref.n, m.n)
            buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
            out = Agents.empty(m.n + ref.n + 1)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record(stream)
            nb = eng.aura_encode(m, ref, buf, stream=stream)
            e1.record(stream)
            eng.aura_decode(buf, nb, ref, out, stream=stream)
            e2.record(stream)
            torch.cuda.synchronize()
            plain = eng.aura_encode(m, empty, torch.empty(eng.aura_max_size(0, m.n),
                                                          dtype=torch.uint8, device="cuda"),
                                    stream=stream)
            assert out.n == m.n
            rows.append({"step": t + 1, "aura_agents": m.n, "raw_bytes": 40 * m.n,
                         "stream_bytes": nb, "lz4_only_bytes": plain,
                         "encode_ms": round(e0.elapsed_time(e1), 4),
                         "decode_ms": round(e1.elapsed_time(e2), 4)})
    enc_ms = sum(r["encode_ms"] for r in rows)
    n_tot = sum(r["aura_agents"] for r in rows)
    line = _common(n_tot / (enc_ms * 1e-3), enc_ms / len(rows), ws, args,
                   {"workload": "cfg2 slab aura (R = 12 um each side of x = side/2), row f3",
                    "reference": "aura at the last warm-up step, kept for all timed steps",
                    "per_step": rows,
                    "ratio_raw_over_stream": round(sum(r["raw_bytes"] for r in rows) /
                                                   sum(r["stream_bytes"] for r in rows), 3),
                    "ratio_raw_over_lz4_only": round(sum(r["raw_bytes"] for r in rows) /
                                                     sum(r["lz4_only_bytes"] for r in rows), 3)},
                   clk.summary(), eng.stats()["launches"] - launches0, dtype="u8")
    line["metric"] = "aura agents encoded/s (delta + LZ4, device timed)"
    line["unit"] = "agents/s"
    line["roofline"] = None
    line["note"] = "timed region: bdm_aura_encode per step (decode timed alongside); one warp per 1 KB LZ4 chunk"
    print(json.dumps(line), flush=True)


def asdict_safe(cfg):
    from dataclasses import asdict
    return asdict(cfg)


def _onco_ages(n, seed, max_age):
    """Reading R44 ages on the host: the product's own Philox4x32-10 in numpy (the oracle
    is test infrastructure and is not called here)."""
    import numpy as np
    import torch
    ids = np.arange(n, dtype=np.uint64)
    c0, c1 = (ids & 0xFFFFFFFF).astype(np.uint32), (ids >> 32).astype(np.uint32)
    c2 = np.full(n, 0xFFFFFFFC, np.uint32)
    c3 = np.full(n, 2, np.uint32)
    k0, k1 = np.uint32(seed & 0xFFFFFFFF), np.uint32(seed >> 32)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0.astype(np.uint64)
        p1 = np.uint64(0xCD9E8D57) * c2.astype(np.uint64)
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), p0.astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), p1.astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = np.uint32((int(k0) + 0x9E3779B9) & 0xFFFFFFFF)
        k1 = np.uint32((int(k1) + 0xBB67AE85) & 0xFFFFFFFF)
    age = np.floor(c0.astype(np.float64) * 2.0 ** -32 * max_age).astype(np.int32)
    return torch.from_numpy(age)


def _slab_population(eng, a, cfg, strong, ws, rank, lo, hi, stream):
    """This rank's agents: (strong) the slab's share of the one cfg5 cube, every rank
    drawing the same per-id population (A48); (weak) one cfg2 cube per rank, shifted
    to the rank's x-slab."""
    import torch
    from paper_2503_10796_b200 import Agents
    if strong and ws == 1:  # the whole cube on one GPU (178 GB: no staging buffer)
        eng.init_spheres(a, cfg.n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, stream=stream)
    elif strong:
        chunk = 50_000_000
        tmp = Agents.empty(chunk)
        a.n = 0
        for id0 in range(0, cfg.n, chunk):
            m = min(chunk, cfg.n - id0)
            eng.init_spheres(tmp, m, id0=id0, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo,
                             stream=stream)
            torch.cuda.synchronize()
            if ws == 1:
                sel = None
                k = m
            else:
                sel = (tmp.x[:m] >= lo) & (tmp.x[:m] < hi)
                k = int(sel.sum())
            for f in ("x", "y", "z", "diameter", "id", "flags"):
                src = getattr(tmp, f)[:m] if sel is None else getattr(tmp, f)[:m][sel]
                getattr(a, f)[a.n:a.n + k].copy_(src)
            a.n += k
        del tmp
        torch.cuda.empty_cache()
    else:
        eng.init_spheres(a, cfg.n, id0=rank * cfg.n, seed=cfg.seed, side=cfg.side,
                         d_lo=cfg.d_lo, d_width=cfg.d_width, d_random=cfg.d_random,
                         stream=stream)
        torch.cuda.synchronize()
        a.x[:cfg.n] += rank * cfg.side
    torch.cuda.synchronize()


def _slab_phase(args, ws, rank, local, strong, steps, warmup):
    """One x-slab measurement through the C-ABI exchange (bdm_aura_exchange over NCCL,
    or the plain step on one GPU): device time per step (max over ranks), the exchange
    share, and the work counters of one step for the roofline."""
    import torch
    import torch.distributed as dist
    from paper_2503_10796_b200 import Agents, Engine, Params
    from paper_2503_10796_b200.slabs import NativeSlabDomain
    cfg = W.CFG5 if strong else W.CFG2
    side_x = cfg.side if strong else cfg.side * ws
    lo = -math.inf if rank == 0 else rank * side_x / ws
    hi = math.inf if rank == ws - 1 else (rank + 1) * side_x / ws
    n_est = cfg.n // ws if strong else cfg.n
    cap = n_est + 4096 if strong and ws == 1 else int(n_est * 1.15) + 4096
    eng = Engine(local, cap)
    eng.set_option("mech_kernel", args.mech_kernel)
    a = Agents.empty(cap)
    stream = torch.cuda.current_stream(local)
    _slab_population(eng, a, cfg, strong, ws, rank, lo, hi, stream)
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    detect_static=cfg.detect_static)
    uid = None
    if ws > 1:
        obj = [eng.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    elif args.force_slabs:
        uid = bytes(128)  # one rank: the exchange runs (frame only), no NCCL
    if uid is not None:
        dom = NativeSlabDomain([eng], [a], [(lo, hi)], params, stream=stream, uid=uid, rank=rank,
                               nranks=ws, ghost_capacity=int(0.02 * n_est) + 65536)
    else:
        dom = None
    eng.step(a, params, stream=stream, sync=True)  # sizes the grid
    gi = eng.grid_info()
    T = [(d + 3) // 4 + 8 for d in gi["dims"]]
    eng.reserve(0, T[0] * T[1] * T[2] * 64)
    for _ in range(warmup):
        if dom:
            dom.step()
        else:
            eng.step(a, params, stream=stream)
    pst = Params(**{**params.__dict__, "collect_stats": True})
    if dom:
        dom.exchange()
        eng.grid_build(a, params.radius, stream=stream, ghosts=dom.ghosts[0] if dom.ghosts[0].n else None)
        eng.mech_step(a, pst, stream=stream)
    else:
        eng.step(a, pst, stream=stream)
    eng.sync(stream)
    st = eng.stats()
    n_loc = a.n
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.stats()["launches"]
    with ClockSampler(local) as clk:
        e0.record(stream)
        for k in range(steps):
            ev[k][0].record(stream)
            if dom:
                dom.exchange()
            ev[k][1].record(stream)
            g = dom.ghosts[0] if dom and dom.ghosts[0].n else None
            eng.grid_build(a, params.radius, stream=stream, ghosts=g)
            eng.mech_step(a, params, stream=stream)
            ev[k][2].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
    eng.sync(stream)
    x_ms = sum(ev[k][0].elapsed_time(ev[k][1]) for k in range(steps)) / steps
    c_ms = sum(ev[k][1].elapsed_time(ev[k][2]) for k in range(steps)) / steps
    vals = torch.tensor([e0.elapsed_time(e1) / steps, x_ms, c_ms, float(n_loc)],
                        dtype=torch.float64, device="cuda")
    if ws > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = vals[3:4].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    else:
        mx, tot = vals, vals[3:4]
    ms_step = float(mx[0])
    peaks, src = _peaks()
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clocks = clk.summary()
    max_mhz = clocks["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    fp64 = (FP64_PER_CAND * st["cand"] + FP64_PER_NBR * st["nbr"] + FP64_PER_CONT * st["cont"] +
            FP64_PER_AGENT * n_loc)
    fp64_peak = sm_count * 64 * max_mhz * 1e6
    b_alg = (B_ALG_PER_AGENT + (B_ALG_STATIC_EXTRA if cfg.detect_static else 0.0)) * n_loc
    t_roof = max(b_alg / (peaks["hbm_gbs"] * 1e9), fp64 / fp64_peak)
    res = {"ms_per_step": ms_step, "value": float(tot[0]) / (ms_step * 1e-3),
           "agents_total": int(tot[0]), "agents_rank0": n_loc,
           "exchange_ms": float(mx[1]), "compute_ms": float(mx[2]),
           "exchange_share": float(mx[1]) / ms_step if ms_step > 0 else None,
           "ghosts_rank0": dom.ghosts[0].n if dom else 0,
           "roofline_rank0": {"bound": "alu", "t_roof_ms": t_roof * 1e3,
                              "frac_of_step": t_roof * 1e3 / ms_step,
                              "fp64_term_ms": fp64 / fp64_peak * 1e3,
                              "hbm_term_ms": b_alg / (peaks["hbm_gbs"] * 1e9) * 1e3},
           "clocks": clocks, "gpu_launches": eng.stats()["launches"] - launches0}
    if dom is not None and not strong and not args.no_e2e:
        res["e2e"] = _slab_e2e(dom, a, ws, steps)
    del dom, a, eng
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def _slab_e2e(dom, a, ws, steps):
    """End to end through the public API at N GPUs: every rank keeps its slab's state in
    pinned host memory; each step copies it to the device, runs the whole step
    (bdm_aura_exchange + bdm_grid_build + bdm_mech_step) and copies the new state back.
    Host clock around each synchronized step, max over ranks."""
    import torch
    import torch.distributed as dist
    fields = ("x", "y", "z", "diameter", "id", "flags")
    host = {f: torch.empty(getattr(a, f).shape, dtype=getattr(a, f).dtype, pin_memory=True)
            for f in fields}
    n = a.n
    for f in fields:
        host[f][:n].copy_(getattr(a, f)[:n])
    torch.cuda.synchronize()
    times, h2d, d2h = [], 0, 0
    for _ in range(steps):
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for f in fields:
            getattr(a, f)[:n].copy_(host[f][:n], non_blocking=True)
        a.n = n
        dom.step()
        n2 = a.n
        if n2 > host["x"].numel():  # the slab grew past the host copy: stop measuring
            break
        for f in fields:
            host[f][:n2].copy_(getattr(a, f)[:n2], non_blocking=True)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        h2d += 40 * n
        d2h += 40 * n2
        n = n2
    k = len(times)
    t = torch.tensor([statistics.median(times) if k else float("nan"), float(n)],
                     dtype=torch.float64, device="cuda")
    tmax = t[0:1].clone()
    tot = t[1:2].clone()
    if ws > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms = float(tmax[0]) * 1e3
    return {"value": float(tot[0]) / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d // max(k, 1), "d2h_bytes_per_step": d2h // max(k, 1),
            "ms_per_step": ms, "steps": k,
            "timing": "host clock around each synchronized step, median, max over ranks",
            "api": "per rank: pinned host SoA -> device, bdm_aura_exchange + bdm_grid_build + "
                   "bdm_mech_step, device -> host (rank 0's bytes)"}


def run_slabs(args, ws, rank, local):
    """x-slab decomposition over N GPUs through the C-ABI exchange
    (bdm_dist_init / bdm_aura_exchange over NCCL, one rank per GPU).  The line is the
    weak-scaled cfg2 workload (one 10M-agent cfg2 cube per GPU, slabs side by side in
    x); strong_cfg5 is the 1.7B-agent cfg5 cube split into N slabs (the north_star's
    scaling target: S_N = T_1 / T_N with T_1 from the N = 1 line's strong_cfg5).
    --python-protocol (or --aura-codec) runs the reference protocol of slabs.py."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.python_protocol or args.aura_codec:
        return run_slabs_python(args, ws, rank, local)
    strong_only = args.config == "cfg5"
    weak = None if strong_only else _slab_phase(args, ws, rank, local, False, args.steps, args.warmup)
    strong = None
    if strong_only or args.strong_steps > 0:
        try:
            strong = _slab_phase(args, ws, rank, local, True,
                                 args.steps if strong_only else args.strong_steps,
                                 args.warmup if strong_only else 2)
        except Exception as e:  # noqa: BLE001 (reported in the line)
            strong = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0:
        main = weak if weak is not None else strong
        line = _common(main["value"], main["ms_per_step"], ws, args,
                       {"workload": ("cfg5 (configs[4]) x-slabs" if weak is None
                                     else "cfg2 (configs[1]) per GPU, x-slabs side by side"),
                        "agents_total": main["agents_total"], "slabs": ws,
                        "transport": "bdm_aura_exchange (C ABI, NCCL p2p + all-reduce)"
                        if ws > 1 else "none (one slab)",
                        "l2": "inputs larger than L2; no flush", "parallelism": f"x-slab {ws}"},
                       main["clocks"], main["gpu_launches"])
        line["scaling"] = "strong" if weak is None else "weak"
        line["roofline"] = {"bound": "alu", "kernel": "rank 0's step (grid + mechanics)",
                            **main["roofline_rank0"]}
        line["exchange"] = {k: main[k] for k in ("exchange_ms", "compute_ms", "exchange_share",
                                                 "ghosts_rank0", "agents_rank0")}
        line["e2e"] = main.get("e2e")
        if line["e2e"] is None:
            line["e2e_note"] = "not measured (--no-e2e, or the strong cfg5 line: no host staging)"
        if weak is not None and strong is not None:
            line["strong_cfg5"] = strong
        line["note"] = "device-timed, max over ranks, of the whole step (exchange + grid + mechanics)"
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_slabs_python(args, ws, rank, local):
    """The reference protocol (slabs.py SlabDomain over torch.distributed), kept for the
    row-f3 aura codec and as a cross-check of the C path."""
    import torch
    import torch.distributed as dist
    from paper_2503_10796_b200 import Agents, Engine, Params
    from paper_2503_10796_b200.slabs import DistTransport, LibOps, Slab, SlabDomain
    strong = args.config == "cfg5"
    cfg = W.CFG5 if strong else W.CFG2
    n_local_est = cfg.n // ws if strong else cfg.n
    side_x = cfg.side if strong else cfg.side * ws
    lo = -math.inf if rank == 0 else rank * side_x / ws
    hi = math.inf if rank == ws - 1 else (rank + 1) * side_x / ws
    cap = int(n_local_est * 1.15) + 4096
    eng = Engine(local, cap)
    a = Agents.empty(cap)
    stream = torch.cuda.current_stream(local)
    _slab_population(eng, a, cfg, strong, ws, rank, lo, hi, stream)
    ops = LibOps(eng, stream=stream)
    tr = DistTransport(ops, torch.device("cuda", local)) if ws > 1 else None
    if tr is None:
        from paper_2503_10796_b200.slabs import LocalTransport
        tr = LocalTransport()
    params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp,
                    detect_static=cfg.detect_static)
    dom = SlabDomain([Slab(rank, lo, hi, ops, a)], tr, params, aura_codec=args.aura_codec)
    for _ in range(args.warmup):
        dom.step()
    n_loc = a.n
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.stats()["launches"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            dom.step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    tot = torch.tensor([float(n_loc)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms_step = float(ms[0]) / args.steps
    value = float(tot[0]) / (ms_step * 1e-3)
    if rank == 0:
        line = _common(value, ms_step, ws, args,
                       {"workload": ("cfg5 (configs[4]) x-slabs" if strong
                                     else "cfg2 (configs[1]) per GPU, x-slabs side by side"),
                        "agents_total": int(tot[0]), "slabs": ws,
                        "transport": "torch.distributed NCCL p2p + all-reduce (slabs.py)" if ws > 1
                        else "local", "aura_codec": bool(args.aura_codec),
                        "l2": "inputs larger than L2; no flush", "parallelism": f"x-slab {ws}"},
                       clk.summary(), eng.stats()["launches"] - launches0)
        line["scaling"] = "strong" if strong else "weak"
        line["roofline"] = None
        line["e2e"] = None
        line["note"] = "reference protocol (slabs.py); device-timed max over ranks"
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def measure_e2e(eng, cfg, params, stream, steps: int = 20):
    """Same metric end to end on a pinned host state: every step copies the agents host
    -> device, runs the step and copies the new state device -> host.  The value is
    bdm_run_host over `steps` steps (the download of step k and the upload of step k+1
    overlap chunk by chunk, full-duplex PCIe: 8.2 ms for both directions at once against
    12.7 ms one after the other, tools/pcie_duplex.py), host clock around the whole call
    (20 steps, so the first upload and the last download, which overlap nothing, weigh
    what they weigh in a long run rather than a seventh of the time each); the
    per-call bdm_step_host median is reported next to it.  The warm-up call sorts the
    host arrays into the grid order; the timed steps run in place with option
    sort_every = 0 (row f1), so the order stays and only x, y, z, flags come back (d and
    id do not change in a step)."""
    import torch
    from paper_2503_10796_b200 import Agents
    n = cfg.n
    hin = Agents.empty(n, pin=True)
    hout = Agents.empty(n, pin=True)
    dev = Agents.empty(n)
    eng.init_spheres(dev, n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                     d_random=cfg.d_random, stream=stream)
    torch.cuda.synchronize()
    for k in ("x", "y", "z", "diameter", "id", "flags"):
        getattr(hin, k).copy_(getattr(dev, k))
    hin.n = n
    eng.set_option("sort_every", 1)
    eng.step_host(hin, hout, dev, params, stream=stream)  # warm-up: sorts into hout
    torch.cuda.synchronize()
    eng.set_option("sort_every", 0)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        eng.step_host(hout, hout, dev, params, stream=stream)  # synchronizing
        times.append(time.perf_counter() - t0)
    dt_call = statistics.median(times)
    eng.run_host(hout, dev, params, 2, stream=stream)  # warm-up of the pipelined path
    t0 = time.perf_counter()
    eng.run_host(hout, dev, params, steps, stream=stream)  # synchronizing
    dt = (time.perf_counter() - t0) / steps
    eng.set_option("sort_every", 1)
    bi = n * (4 * 8 + 2 * 4)
    bo = n * (3 * 8 + 4)
    # the PCIe floor: the same bytes copied alone (pinned host <-> device, same stream)
    tr = []
    for _ in range(3):
        t0 = time.perf_counter()
        for f in ("x", "y", "z", "diameter", "id", "flags"):
            getattr(dev, f)[:n].copy_(getattr(hout, f)[:n], non_blocking=True)
        for f in ("x", "y", "z", "flags"):
            getattr(hout, f)[:n].copy_(getattr(dev, f)[:n], non_blocking=True)
        torch.cuda.synchronize()
        tr.append(time.perf_counter() - t0)
    t_copy = statistics.median(tr)
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
            "ms_per_step": dt * 1e3, "steps": steps,
            "step_host_ms": dt_call * 1e3,
            "step_host_ms_all": [round(t * 1e3, 3) for t in times],
            "copy_only_ms": t_copy * 1e3,
            "copy_gbs": (bi + bo) / t_copy / 1e9,
            "note": "copy_only_ms = the same bytes copied one way after the other; "
                    "bdm_run_host overlaps step k's download with step k+1's upload",
            "timing": "host clock around one bdm_run_host call of `steps` steps (synchronizing)",
            "api": "bdm_run_host (C ABI, pinned host buffers, in place, sort_every 0, 8 chunks)"}


def cpu_baseline(cfg=W.CFG2):
    """cpu_baseline of a mechanics line: whole oracle steps of the config on all host
    cores (cfg1: 10 steps; cfg2: one 10M-agent step; cfg5: one step of a 10M-agent cube
    of the cfg5 population, the 1.7B agents do not fit the host)."""
    if cfg.name == "cfg5":
        sub = W.MechConfig("cfg5 (10M-agent cube)", 10_000_000,
                           W.side_for_fraction(10_000_000, 1000.0, 0.5), cfg.d_lo, 0.0, False,
                           cfg.steps, cfg.detect_static)
        return cpu_baseline_mech(sub, steps=1, note="; a 10M-agent cube of the cfg5 population "
                                 "(same density and diameter) stands in for the 1.7B agents")
    if cfg.name == "cfg1":
        return cpu_baseline_mech(cfg, steps=10)
    return cpu_baseline_mech(cfg, steps=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(W.PRESETS) + ["aura"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mech-kernel", type=int, default=5,
                    help="5 tile7 (default), 0 tile6, 1 per-agent reference, 4 row-broadcast")
    ap.add_argument("--tile-depth", type=int, default=0,
                    help="tile work unit: 0 auto (by agents per box), 1 or 2 tiles deep")
    ap.add_argument("--tile-order", type=int, default=0,
                    help="row f1: 0 row-major tiles, 1 blocked Hilbert")
    ap.add_argument("--sort-every", type=int, default=1,
                    help="row f1: reorder the agents every K-th step (0 = never)")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the x-slab protocol path even on one GPU (a check of that path)")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: seconds the oracle's --steps K --warmup W should take")
    ap.add_argument("--no-graph", action="store_true",
                    help="skip the CUDA-graph replay measurement of the step")
    ap.add_argument("--python-protocol", action="store_true",
                    help="x-slabs through the reference protocol of slabs.py (not the C ABI)")
    ap.add_argument("--strong-steps", type=int, default=3,
                    help="steps of the strong-scaled cfg5 x-slab measurement added to the "
                         "N-GPU line (and T_1 to the N = 1 line); 0 skips it")
    ap.add_argument("--aura-codec", action="store_true",
                    help="row f3: x-slab aura as delta + LZ4 streams (links slower than NVLink)")
    ap.add_argument("--shuffle", action="store_true",
                    help="start from a random memory order of the agents (row f1 sweeps)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
