"""Builds paper_2503_10796_b200/libbdm.so (sm_100a) in-tree with nvcc.

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source view),
-fmad=false (no implicit a*b+c contraction: the explicit fma() calls are the only
fused sites, reading R9), IEEE division and square root (nvcc defaults without
--use_fast_math).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbdm.so")
SOURCES = ["bdm_abi.cu", "kernels_grid.cu", "kernels_mech.cu", "kernels_divide.cu",
           "kernels_sir.cu", "kernels_slab.cu", "kernels_diffusion.cu", "kernels_onco.cu",
           "kernels_aura.cu", "kernels_row.cu", "dist_abi.cu"]
HEADERS = ["bdm_internal.cuh", "mech_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
] + os.environ.get("BDM_NVCC_EXTRA", "").split()  # experiments only (A/B variants)


def _newest_input() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "bdm.h"))
    return max(os.path.getmtime(f) for f in files)


STAMP = SO + ".cmd"  # the full nvcc command of the built library (variants rebuild)


def _command(out: str) -> list:
    return [NVCC, *NVCC_FLAGS, "-shared", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
            *[os.path.join(CSRC, f) for f in SOURCES], "-o", out, "-lcudart"]


def _stamp_text() -> str:
    return " ".join(_command(SO))


def up_to_date() -> bool:
    """The library exists, is newer than every source, and was built by this exact
    command (flags included: an A/B variant built with BDM_NVCC_EXTRA is not reused)."""
    if not (os.path.exists(SO) and os.path.exists(STAMP)):
        return False
    if os.path.getmtime(SO) < _newest_input():
        return False
    with open(STAMP) as f:
        return f.read() == _stamp_text()


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc -c per source, in parallel, then one nvcc -shared link."""
    if not force and up_to_date():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

    def compile_one(f):
        obj = os.path.join(objdir, f.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, *inc, "-c", os.path.join(CSRC, f), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return f, cmd, r, obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = os.path.join(HERE, "build.log")
    tmp = SO + ".tmp"
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
            *[o for _, _, _, o in results], "-o", tmp, "-lcudart"]
    with open(log, "w") as f:
        for name, cmd, r, _ in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    bad = [(n, r) for n, _, r, _ in results if r.returncode != 0]
    if bad:
        for n, r in bad:
            sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed for {[n for n, _ in bad]} (see {log})")
    res = subprocess.run(link, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(link) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc link failed (see {log})")
    if verbose:
        with open(log) as f:
            sys.stderr.write(f.read())
    os.replace(tmp, SO)
    with open(STAMP, "w") as f:
        f.write(_stamp_text())
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
