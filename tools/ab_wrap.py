"""A/B against the committed mechanics kernel: `python tools/ab_wrap.py on` snapshots
HEAD's kernels_mech.cu to tools/ab_base/ (git-ignored) and wraps the working copy so that
-DBDM_BASELINE builds the snapshot; `off` removes the wrapper again (before a commit)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2503_10796_b200", "csrc", "kernels_mech.cu")
BASE = os.path.join(ROOT, "tools", "ab_base", "kernels_mech_base.cu")
HEAD = '#ifdef BDM_BASELINE\n#include "../../tools/ab_base/kernels_mech_base.cu"\n#else\n'
TAIL = '#endif  // BDM_BASELINE\n'

s = open(SRC).read()
wrapped = s.startswith(HEAD)
if wrapped:
    s = s[len(HEAD):-len(TAIL)]
if sys.argv[1] == "on":
    os.makedirs(os.path.dirname(BASE), exist_ok=True)
    base = subprocess.run(["git", "show", "HEAD:paper_2503_10796_b200/csrc/kernels_mech.cu"],
                          cwd=ROOT, capture_output=True, text=True, check=True).stdout
    open(BASE, "w").write(base)
    s = HEAD + s + TAIL
open(SRC, "w").write(s)
print("wrapped" if sys.argv[1] == "on" else "unwrapped")
