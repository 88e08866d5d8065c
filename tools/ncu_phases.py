"""Instructions and stall samples of the tile7 kernel by phase (line ranges of
kernels_mech.cu): python tools/ncu_phases.py rep name:line,name:line,..."""
import csv
import subprocess
import sys

rep, spec = sys.argv[1], sys.argv[2]
n_agents = float(sys.argv[3]) if len(sys.argv) > 3 else 1e7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, cur, f = {}, None, ""
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed", 3)
        iss = r.index("Warp Stall Sampling (All Samples)", 3)
        hdr = r
        continue
    if r[0] != "":
        cur = (f, int(r[0]))
        continue
    try:
        n, s = int(r[ie]), int(r[iss])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0, {}])
    a[0] += n
    a[1] += s
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "(Not" not in name:
            try:
                a[2][name] = a[2].get(name, 0) + int(r[k])
            except ValueError:
                pass
marks = sorted((int(x.split(":")[1]), x.split(":")[0]) for x in spec.split(","))
tot = sum(v[1] for v in agg.values())
toti = sum(v[0] for v in agg.values())
print(f"total {toti / n_agents:.1f} warp-instr/agent, {tot} samples")
for i, (lo, name) in enumerate(marks):
    hi = marks[i + 1][0] if i + 1 < len(marks) else 10 ** 9
    n = s = 0
    st = {}
    for (ff, l), (a, b, c) in agg.items():
        if ff == "kernels_mech.cu" and lo <= l < hi:
            n += a
            s += b
            for k, v in c.items():
                st[k] = st.get(k, 0) + v
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    print(f"{name:10s} {lo:5d} {n / n_agents:6.1f}/agent  samples {100 * s / tot:5.1f}%  " +
          " ".join(f"{k[6:]}={100 * v / tot:.1f}" for k, v in top))
n = s = 0
for (ff, l), (a, b, c) in agg.items():
    if ff != "kernels_mech.cu":
        n += a
        s += b
print(f"other files {n / n_agents:.1f}/agent samples {100 * s / tot:.1f}%")
