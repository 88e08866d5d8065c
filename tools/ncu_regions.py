"""Per-region SASS breakdown of an ncu report: python tools/ncu_regions.py rep [chunk]"""
import csv, subprocess, sys
rep = sys.argv[1]; chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ie = h.index('Instructions Executed'); its = h.index('Warp Stall Sampling (All Samples)'); isrc = h.index('Source'); ith = h.index('Avg. Threads Executed')
tot = sum(int(r[ie]) for r in data); tots = sum(int(r[its]) for r in data)
print(f"total warp-inst {tot/1e6:.1f}M  stall samples {tots}")
for i in range(0, len(data), chunk):
    c = sum(int(r[ie]) for r in data[i:i+chunk]); s = sum(int(r[its]) for r in data[i:i+chunk])
    th = sum(int(r[ie]) * float(r[ith]) for r in data[i:i+chunk]) / max(c, 1)
    if c > tot * 0.01 or s > tots * 0.015:
        ops = [r[isrc].split()[1] if r[isrc].strip().startswith('@') else r[isrc].split()[0] for r in data[i:i+chunk]]
        print(f"{i:5d} {c/1e6:8.1f}M ({c/tot*100:4.1f}%) thr={th:4.1f} stall={s/tots*100:4.1f}%  {' '.join(o for o in ops if o.startswith(('D','F','LDS','STS','LDG','BAR','MUFU','SHFL')))[:100]}")
