import math, sys, numpy as np
sys.path.insert(0, '.')
import oracle as orc
from paper_2503_10796_b200 import Agents, Engine, Params
V_MAX = (math.pi / 6.0) * 1728.0
for kern in (0, 1):
    e = Engine(0, 1 << 16); e.set_option("mech_kernel", kern)
    n = 257; side = 1000.0 * (n / 1e6) ** (1 / 3)
    o = orc.init_spheres(n, 1, side, 8.0); o["vol"] = orc.init_volumes(o)
    a = Agents.from_numpy(o, capacity=n * 64)
    gp = Params(seed=1, collect_stats=True); op = orc.mech_params()
    for t in range(8):
        gp.step = t
        pre = a.numpy()
        e.step(a, gp)
        st = e.stats()
        mid = a.numpy()
        e.grow_divide(a, gp, 400.0, V_MAX)
        om, cnt = orc.mech_step(pre, op)
        o, _ = orc.cfg3_step(o, op, 400.0, V_MAX, 1, t)
        g = a.numpy()
        gi = np.argsort(g["id"]); oi = np.argsort(o["id"])
        dx = np.abs(g["x"][gi] - o["x"][oi])
        # mechanics-only comparison on the same input
        mi = np.argsort(mid["id"]); pi = np.argsort(pre["id"])
        dm = np.abs(mid["x"][mi] - om["x"][pi])
        print(kern, t, len(g["x"]), "final maxdiff", dx.max(), "n_bad", int((dx > 0).sum()),
              "| mech-only n_bad", int((dm > 0).sum()), "stats", st["cand"], cnt["cand"], st["nbr"], cnt["nbr"], st["cont"], cnt["cont"])
