"""Debug: compare mech kernels 0 / 4 against the oracle on the failing edge cases."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as orc, workloads as W
from paper_2503_10796_b200 import Engine, Agents, Params

def run(kernel, s, gp):
    e = Engine(0, 1 << 13); e.set_option("mech_kernel", kernel); e.set_option("fuse_reduce", 1)
    a = Agents.from_numpy(s); e.step(a, gp, sync=True); g = a.numpy(); e.close(); return g

def cmp(name, s, gp, op):
    o, _ = orc.step_full(s, op)
    for k in (0, 4):
        g = run(k, s, gp)
        bad = [f for f in ("id", "x", "y", "z", "flags") if not np.array_equal(g[f], o[f])]
        print(name, "kernel", k, "bad fields", bad)
        if bad:
            ids = o["id"]; pos = {int(i): j for j, i in enumerate(g["id"])}
            diff = [int(i) for j, i in enumerate(ids) if int(i) not in pos or g["x"][pos[int(i)]] != o["x"][j]]
            print("  n differing", len(diff), diff[:10])
            print("  gpu ids head", g["id"][:8], "orc", o["id"][:8])

s = orc.init_spheres(2000, 4, 50.0, 10.0)
gp = Params(dt=1.0, boundary=1, lo=(5, 5, 5), hi=(45, 45, 45))
op = orc.mech_params(dt=1.0, boundary=1, lo=(5, 5, 5), hi=(45, 45, 45))
cmp("closed", s, gp, op)
gp = Params(dt=1.0); op = orc.mech_params(dt=1.0)
cmp("open-dense", s, gp, op)
s = orc.init_spheres(3000, 2, 40.0, 10.0)
cmp("cap", s, gp, op)
rng = np.random.default_rng(5)
for n in (300, 1500):
    for dmode in ("tiny", "wide"):
        d = rng.uniform(0.5, 2.0, n) if dmode == "tiny" else rng.choice([2.0, 30.0], n)
        side = (n * np.mean(d) ** 3 / 0.5) ** (1 / 3)
        p = rng.uniform(0, side, (n, 3))
        s = {"x": p[:, 0].copy(), "y": p[:, 1].copy(), "z": p[:, 2].copy(), "d": d,
             "id": np.arange(n, dtype=np.uint32), "flags": np.zeros(n, np.uint32)}
        cmp(f"{dmode}{n}", s, Params(), orc.mech_params())
