"""PCIe copy bandwidth: H2D alone, D2H alone, and both at once on two streams (pinned)."""
import time
import torch

n_up, n_dn = 400 << 20, 280 << 20
hu = torch.empty(n_up, dtype=torch.uint8).pin_memory()
hd = torch.empty(n_dn, dtype=torch.uint8).pin_memory()
du = torch.empty(n_up, dtype=torch.uint8, device="cuda")
dd = torch.empty(n_dn, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, k=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


def up():
    with torch.cuda.stream(s1):
        du.copy_(hu, non_blocking=True)


def dn():
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)


def both():
    up()
    dn()


a, b, c = t(up), t(dn), t(both)
print(f"H2D {n_up / a / 1e6:.1f} GB/s ({a:.2f} ms)  D2H {n_dn / b / 1e6:.1f} GB/s ({b:.2f} ms)  "
      f"both {c:.2f} ms (sequential would be {a + b:.2f})")
