import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as orc
from paper_2503_10796_b200 import Engine, Agents, Params

def analyse(name, s, prm, opts):
    n = len(s["x"])
    e = Engine(0, 1 << 13); e.set_option("mech_kernel", 4)
    for k, v in opts: e.set_option(k, v)
    a = Agents.from_numpy(s); e.step(a, prm, sync=True); g = a.numpy()
    gi = e.grid_info()
    e0 = Engine(0, 1 << 13); a0 = Agents.from_numpy(s); e0.step(a0, prm, sync=True); g0 = a0.numpy()
    L = gi["L"]; o = gi["origin"]
    f = g["flags"].astype(np.int64)
    marked = (f >> 31) == 1
    paths = {}
    for slot in range(n):
        key = (int((f[slot] >> 8) & 0x7fffff), int(f[slot] & 255)) if marked[slot] else (-1, -1)
        ok = g["id"][slot] == g0["id"][slot]
        paths.setdefault(key, [0, 0])[0 if ok else 1] += 1
    print(name, opts, "dims", gi["dims"], "marked", int(marked.sum()), "of", n)
    for k in sorted(paths): print("   tile,path", k, "ok/bad", paths[k])

rng = np.random.default_rng(5)
n = 1500
d = rng.choice([2.0, 30.0], n)
side = (n * np.mean(d) ** 3 / 0.5) ** (1 / 3)
p = rng.uniform(0, side, (n, 3))
s = {"x": p[:, 0].copy(), "y": p[:, 1].copy(), "z": p[:, 2].copy(), "d": d,
     "id": np.arange(n, dtype=np.uint32), "flags": np.zeros(n, np.uint32)}
analyse("wide", s, Params(), (("prefilter", 9),))
analyse("wide-nodense", s, Params(), (("prefilter", 9), ("dense", 0)))
s = orc.init_spheres(2000, 4, 50.0, 10.0)
analyse("open-dense", s, Params(dt=1.0), (("prefilter", 9),))
