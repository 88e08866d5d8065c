"""Run bdm_diffuse (TMA path) once on one grid shape; exit 0 if it ran and matched."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2503_10796_b200 import CGrid3, Engine
import oracle as orc

nx, ny, nz = (int(v) for v in sys.argv[1:4])
e = Engine(0, 16)
u0 = np.random.default_rng(1).uniform(0, 1, (nz, ny, nx))
u = torch.from_numpy(u0).cuda()
v = torch.empty_like(u)
e.diffuse(u, v, CGrid3.make(nx, ny, nz, (0, 0, 0), 1.0), 0.1, 0.0, 0.5)
torch.cuda.synchronize()
ok = np.array_equal(v.cpu().numpy(), orc.diffuse(u0, orc.Grid3(nx, ny, nz), 0.1, 0.0, 0.5, 1))
print(nx, ny, nz, "match" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
