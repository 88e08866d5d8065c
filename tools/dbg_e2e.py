"""bdm_run_host chunk-count sweep at cfg2 (10M agents): ms per end-to-end step."""
import sys, time
sys.path.insert(0, ".")
import torch
import workloads as W
from paper_2503_10796_b200 import Agents, Engine, Params
cfg = W.CFG2
n = cfg.n
eng = Engine(0, n)
stream = torch.cuda.Stream()
dev = Agents.empty(n)
eng.init_spheres(dev, n, seed=cfg.seed, side=cfg.side, d_lo=cfg.d_lo, d_width=cfg.d_width,
                 d_random=cfg.d_random, stream=stream)
torch.cuda.synchronize()
h = Agents.empty(n, pin=True)
for k in ("x", "y", "z", "diameter", "id", "flags"):
    getattr(h, k).copy_(getattr(dev, k))
h.n = n
params = Params(k=cfg.k, gamma=cfg.gamma, dt=cfg.dt, max_displacement=cfg.max_disp, detect_static=True)
eng.set_option("sort_every", 1)
eng.step_host(h, h, dev, params, stream=stream)
eng.set_option("sort_every", 0)
for chunks in (1, 4, 8, 16, 32, 64):
    eng.run_host(h, dev, params, 2, chunks=chunks, stream=stream)
    t0 = time.perf_counter()
    eng.run_host(h, dev, params, 7, chunks=chunks, stream=stream)
    print("chunks", chunks, "ms/step", round((time.perf_counter() - t0) / 7 * 1e3, 3), flush=True)
# copies alone, both directions concurrently on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    for f in ("x", "y", "z", "diameter", "id", "flags"):
        getattr(dev, f)[:n].copy_(getattr(h, f)[:n], non_blocking=True)
with torch.cuda.stream(s2):
    tmp = Agents.empty(n, pin=True)
    for f in ("x", "y", "z", "flags"):
        getattr(tmp, f)[:n].copy_(getattr(dev, f)[:n], non_blocking=True)
torch.cuda.synchronize()
print("h2d || d2h alone ms", round((time.perf_counter() - t0) * 1e3, 3))
t0 = time.perf_counter()
for f in ("x", "y", "z", "diameter", "id", "flags"):
    getattr(dev, f)[:n].copy_(getattr(h, f)[:n], non_blocking=True)
torch.cuda.synchronize()
print("h2d alone ms", round((time.perf_counter() - t0) * 1e3, 3))
t0 = time.perf_counter()
for f in ("x", "y", "z", "flags"):
    getattr(tmp, f)[:n].copy_(getattr(dev, f)[:n], non_blocking=True)
torch.cuda.synchronize()
print("d2h alone ms", round((time.perf_counter() - t0) * 1e3, 3))
