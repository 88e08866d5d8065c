#!/bin/bash
# A/B of a compile-time variant: bash tools/gpu_abx.sh "-DFLAG ..." [cfg3]
# A = default build, B = build with the flags; tile-kernel parity tests and cfg2 benches
# (and the cfg3 run when the second argument is cfg3) for both.
mkdir -p gpurun_out
for v in A B; do
  if [ $v = B ]; then X="$1"; else X=""; fi
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_$v.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_sfc.py -q -x -k "not reference and not tile_v1" > gpurun_out/pytest_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/pytest_$v.log)"
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v$r.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bench_$v$r.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4))"
  done
  if [ "$2" = cfg3 ]; then
    timeout 300 python bench.py --config cfg3 --steps 20 --warmup 3 > gpurun_out/bench_cfg3_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bench_cfg3_$v.json').read().strip().splitlines()[-1]); print('$v cfg3', round(sum(p['ms'] for p in d['config']['per_step']),1))"
  fi
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
