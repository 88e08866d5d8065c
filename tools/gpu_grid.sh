#!/bin/bash
# ncu --set full of the cfg2 grid-build kernels (rows a2-a4), after a plain run exits 0.
O=gpurun_out/grid; mkdir -p $O
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1; echo plain=$?
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_key|k_scatter|k_fix_gather' -s 9 -c 3 -o $O/prof_grid python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1; echo ncu=$?
ncu -i $O/prof_grid.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null; echo raw=$?
