#!/bin/bash
# ncu --set full of the f2 (oncology), f3 (aura codec) and a10 (division) kernels, each
# after the same bench command exits 0 without ncu.
O=gpurun_out/rows; mkdir -p $O
B="--no-e2e --no-cpu-baseline"
python bench.py --config onco --steps 3 --warmup 3 $B > $O/onco.json 2>&1; echo onco=$?
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_onco' -s 3 -c 3 -o $O/prof_onco python bench.py --config onco --steps 2 --warmup 3 $B > $O/ncu_onco.log 2>&1; echo ncu_onco=$?
python bench.py --config aura --steps 3 --warmup 3 $B > $O/aura.json 2>&1; echo aura=$?
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_lz4|k_aura' -s 12 -c 6 -o $O/prof_aura python bench.py --config aura --steps 1 --warmup 3 $B > $O/ncu_aura.log 2>&1; echo ncu_aura=$?
for r in onco aura; do ncu -i $O/prof_$r.ncu-rep --page raw --csv > $O/raw_$r.csv 2>/dev/null; done
