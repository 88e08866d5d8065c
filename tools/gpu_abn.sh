#!/bin/bash
# A/B/C...: bash tools/gpu_abn.sh "" "-DFLAG1" "-DFLAG2" ...; tile parity tests + 2 cfg2 benches each
mkdir -p gpurun_out
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_v$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_sfc.py -q -x -k "not reference and not tile_v1" > gpurun_out/pytest_v$i.log 2>&1
  echo "v$i [$X] tests: $(tail -1 gpurun_out/pytest_v$i.log)"
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v$i$r.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bench_v$i$r.json').read().strip().splitlines()[-1]); print('v$i', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
  done
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
