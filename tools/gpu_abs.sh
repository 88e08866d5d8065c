#!/bin/bash
# SIR A/B: bash tools/gpu_abs.sh "" "-DFLAG"; SIR parity tests + cfg4 bench (2 runs)
mkdir -p gpurun_out
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_s$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_sir.py -q -x > gpurun_out/pytest_s$i.log 2>&1
  echo "s$i [$X] tests: $(tail -1 gpurun_out/pytest_s$i.log)"
  for r in 1 2; do
    timeout 300 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_s$i$r.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bench_cfg4_s$i$r.json').read().strip().splitlines()[-1]); print('s$i', round(d['ms_per_step'],4))"
  done
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
