#!/bin/bash
# dense-kernel A/B: bash tools/gpu_abd.sh "" "-DFLAG"; dense parity tests + cfg3
mkdir -p gpurun_out
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_d$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_cfg3.py -q -x -k "dense or cfg3" > gpurun_out/pytest_d$i.log 2>&1
  echo "d$i [$X] tests: $(tail -1 gpurun_out/pytest_d$i.log)"
  timeout 300 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_d$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg3_d$i.json').read().strip().splitlines()[-1]); ps=d['config']['per_step']; print('d$i cfg3', round(sum(p['ms'] for p in ps),1), [round(p['ms'],1) for p in ps[-4:]])"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
