#!/bin/bash
# session 4: grid-build A/B (BDM_NVCC_EXTRA variants): grid parity tests for each variant, two cfg2 bench lines
O=gpurun_out/s4h; mkdir -p $O
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build_v$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_sfc.py -m gpu -q -x -p no:cacheprovider -k "tile7 or sfc" > $O/pytest_v$i.log 2>&1
  echo "v$i [$X] tests: $(tail -1 $O/pytest_v$i.log)"
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 > $O/bench_v$i$r.json 2> $O/bench_v$i$r.err
    python -c "import json; d=json.loads(open('$O/bench_v$i$r.json').read().strip().splitlines()[-1]); print('v$i [$X]', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
  done
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build.log 2>&1
