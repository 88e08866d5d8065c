"""Summary of an ncu --set full report (one kernel launch): duration, DRAM bytes,
occupancy, issue, fp64 pipe, shared-memory wavefronts and the top warp stalls.
python tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}
print(f"  Kernel Name{'':60s} {vals[col['Kernel Name']]}")
for m in METRICS:
    if m in col:
        print(f"  {m:70s} {vals[col[m]]} {units[col[m]]}")
stalls = []
for h, i in col.items():
    if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
       h.startswith("smsp__average_warps_issue_stalled_"):
        if h.endswith("_per_issue_active.ratio"):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            name = h.split("stalled_")[1].replace("_per_issue_active.ratio", "")
            stalls.append((v, name))
for v, name in sorted(stalls, reverse=True)[:8]:
    print(f"  stall {name:30s} {v:.3f}")
