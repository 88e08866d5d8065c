#!/bin/bash
# session 3 A/B of k_sir_update (BDM_NVCC_EXTRA variants): SIR parity tests for the
# first variant, two cfg4 bench lines each
O=gpurun_out/s3d; mkdir -p $O
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build_v$i.log 2>&1
  if [ $i -eq 1 ]; then
    timeout 900 python -m pytest tests/test_gpu_sir.py -m gpu -q -x -p no:cacheprovider > $O/pytest_v$i.log 2>&1
    echo "v$i [$X] tests: $(tail -1 $O/pytest_v$i.log)"
  fi
  for r in 1 2; do
    timeout 300 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_v$i$r.json 2> $O/bench_cfg4_v$i$r.err
    python -c "import json; d=json.loads(open('$O/bench_cfg4_v$i$r.json').read().strip().splitlines()[-1]); print('v$i [$X]', round(d['ms_per_step'],4))"
  done
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build.log 2>&1
