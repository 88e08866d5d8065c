"""Debug: which boxes hold the agents kernel 4 gets wrong."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as orc
from paper_2503_10796_b200 import Engine, Agents, Params

def run(kernel, s, gp, opts=()):
    e = Engine(0, 1 << 13); e.set_option("mech_kernel", kernel); e.set_option("fuse_reduce", 1)
    for k, v in opts: e.set_option(k, v)
    a = Agents.from_numpy(s); e.step(a, gp, sync=True); g = a.numpy(); gi = e.grid_info(); e.close(); return g, gi

def boxes(name, s, gp, opts=()):
    g0, gi = run(0, s, gp)
    g4, _ = run(4, s, gp, opts)
    R = s["d"].max(); L = R * (1 + 2**-20)
    o = [s[c].min() for c in "xyz"]
    byid = {int(i): j for j, i in enumerate(s["id"])}
    bad = np.nonzero((g0["x"] != g4["x"]) | (g0["id"] != g4["id"]))[0]
    bb = {}
    for slot in bad:
        i = int(g0["id"][slot]); j = byid[i]
        b = tuple(int(np.floor((s[c][j] - o[k]) / L)) for k, c in enumerate("xyz"))
        bb[b] = bb.get(b, 0) + 1
    print(name, opts, "dims", gi.get("dims"), "bad slots", len(bad), "first slot", bad[:3], "boxes", sorted(bb.items())[:24], flush=True)

s = orc.init_spheres(2000, 4, 50.0, 10.0)
gp = Params(dt=1.0)
boxes("open-dense", s, gp)
#boxes("open-dense", s, gp, (("dense", 0),))
#boxes("open-dense", s, gp, (("prefilter", 0),))
rng = np.random.default_rng(5)
n = 1500
d = rng.choice([2.0, 30.0], n)
side = (n * np.mean(d) ** 3 / 0.5) ** (1 / 3)
p = rng.uniform(0, side, (n, 3))
s = {"x": p[:, 0].copy(), "y": p[:, 1].copy(), "z": p[:, 2].copy(), "d": d,
     "id": np.arange(n, dtype=np.uint32), "flags": np.zeros(n, np.uint32)}
boxes("wide", s, Params())
#boxes("wide", s, Params(), (("prefilter", 0),))
#boxes("wide-stats", s, Params(collect_stats=True))
boxes("wide-dbg-groupfallback", s, Params(), (("prefilter", 3),))
boxes("wide-dbg-slowrows", s, Params(), (("prefilter", 5),))
s = orc.init_spheres(2000, 4, 50.0, 10.0)
boxes("open-dense-slowrows", s, Params(dt=1.0), (("prefilter", 5),))
boxes("open-dense-groupfb", s, Params(dt=1.0), (("prefilter", 3),))
