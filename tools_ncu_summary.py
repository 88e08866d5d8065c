"""Summarise an ncu report (raw page) for the metrics we track. Usage: python tools_ncu_summary.py rep [kernel-substring]"""
import csv, subprocess, sys
rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__occupancy_limit_shared_mem',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed']
stalls = [x for x in h if x.startswith('smsp__average_warps_issue_stalled_') and x.endswith('_per_issue_active.ratio')]
for row in r[2:]:
    if sub and sub not in row[h.index('Kernel Name')]:
        continue
    for w in want:
        if w in h:
            print(f"  {w:70s} {row[h.index(w)]} {r[1][h.index(w)]}")
    st = sorted(((float(row[h.index(x)] or 0), x) for x in stalls), reverse=True)[:8]
    for v, x in st:
        print(f"  stall {x.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s} {v:.3f}")
    print()
