#!/bin/bash
# session 4: tile7 two-tile units of 672 staged agents, 8 warps x 3 CTAs (depth 3) and
# 4 warps x 4 CTAs (depth 4), against the default (depth 1) at cfg2
O=gpurun_out/s4f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for d in 1 3 4 1 3 4; do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --tile-depth $d > $O/bench_d$d.json 2> $O/bench_d$d.err
  python -c "import json; d=json.loads(open('$O/bench_d$d.json').read().strip().splitlines()[-1]); print('depth $d', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
done
