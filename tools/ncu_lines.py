"""Per-CUDA-source-line breakdown of an ncu report (needs -lineinfo):
python tools/ncu_lines.py rep [file-substring] [min-pct]

Prints, for each source line of the matching file with >= min-pct of the kernel's warp
instructions or stall samples: warp instructions, avg active threads, stall share, text.
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
fsub = sys.argv[2] if len(sys.argv) > 2 else "kernels_mech.cu"
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, lines = None, None, {}
tot_i = tot_s = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed", 3)
        iss = hdr.index("Warp Stall Sampling (All Samples)", 3)
        ith = hdr.index("Avg. Threads Executed", 3)
        continue
    if r[0] == "" and r[2] not in ("", "-"):  # a SASS row under the current line
        try:
            n = int(r[ie]); s = int(r[iss]); th = float(r[ith])
        except ValueError:
            continue
        tot_i += n; tot_s += s
        key = (cur_file, cur_line)
        a = lines.setdefault(key, [0, 0, 0.0, cur_text])
        a[0] += n; a[1] += s; a[2] += n * th
        continue
    if r[0] != "":
        cur_line, cur_text = int(r[0]), r[1]
print(f"total warp-inst {tot_i / 1e6:.1f}M, stall samples {tot_s}")
for (f, ln), (n, s, th, txt) in sorted(lines.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if fsub not in f:
        if n < tot_i * 0.03 and s < tot_s * 0.03:
            continue
    if n >= tot_i * minp / 100 or s >= tot_s * minp / 100:
        print(f"{f.split('/')[-1][:14]:14s}:{ln:5d} {n / 1e6:7.1f}M ({100 * n / tot_i:4.1f}%) "
              f"thr={th / max(n, 1):4.1f} stall={100 * s / max(tot_s, 1):4.1f}%  {txt.strip()[:90]}")

# optional: phase ranges "name:lo-hi,name:lo-hi" (lines of the matching file)
if len(sys.argv) > 4:
    agg = {}
    for spec in sys.argv[4].split(","):
        name, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        for (f, ln), (n, s, th, txt) in lines.items():
            if fsub in f and lo <= ln <= hi:
                a = agg.setdefault(name, [0, 0])
                a[0] += n; a[1] += s
    other_n = tot_i - sum(a[0] for a in agg.values())
    other_s = tot_s - sum(a[1] for a in agg.values())
    for name, (n, s) in list(agg.items()) + [("other", (other_n, other_s))]:
        print(f"  {name:12s} {n / 1e6:8.1f}M ({100 * n / tot_i:4.1f}%)  stall {100 * s / max(tot_s, 1):4.1f}%")
