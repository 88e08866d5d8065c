#!/bin/bash
# cfg5 (one GPU) + cfg2 A/B: bash tools/gpu_ab5.sh "" "-DFLAG"
mkdir -p gpurun_out
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_c$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py -q -x -k "tile and not tile_v1 and not tile_4cta" > gpurun_out/pytest_c$i.log 2>&1
  echo "c$i [$X] tests: $(tail -1 gpurun_out/pytest_c$i.log)"
  timeout 600 python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_c$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg5_c$i.json').read().strip().splitlines()[-1]); print('c$i cfg5', round(d['ms_per_step'],2), round(d['roofline']['mech_ms'],2))"
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2_c$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_c$i.json').read().strip().splitlines()[-1]); print('c$i cfg2', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4))"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
