#!/bin/bash
# session 4: k_zero_counts grid size (blocks per SM), ncu duration of two launches each + one cfg2 bench line
O=gpurun_out/s4s; mkdir -p $O
for b in 16 4 2 1; do
  BDM_NVCC_EXTRA="-DBDM_ZERO_BLOCKS_PER_SM=$b" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build_$b.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_zero_counts -s 5 -c 3 --csv --log-file $O/zero_$b.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_$b.log 2>&1
  echo "blocks/SM $b: $(grep k_zero_counts $O/zero_$b.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') ns"
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 > $O/bench_$b.json 2> $O/bench_$b.err
  python -c "import json; d=json.loads(open('$O/bench_$b.json').read().strip().splitlines()[-1]); print('blocks/SM $b', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build.log 2>&1
