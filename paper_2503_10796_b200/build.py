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
           "kernels_aura.cu"]
HEADERS = ["bdm_internal.cuh"]
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


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= _newest_input():
        return SO
    tmp = SO + ".tmp"
    cmd = [NVCC, *NVCC_FLAGS, "-shared", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, f) for f in SOURCES], "-o", tmp, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
