#!/bin/bash
# A/B: phase 2b one contact per lane (A) vs two interleaved (B: -DBDM_DENSE_ILP2 -DBDM_TILE_ILP2)
mkdir -p gpurun_out
for v in A B; do
  if [ $v = B ]; then X="-DBDM_DENSE_ILP2 -DBDM_TILE_ILP2"; else X=""; fi
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build_$v.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_cfg3.py -q -x -k "not reference and not tile_v1" > gpurun_out/pytest_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/pytest_$v.log)"
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v$r.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bench_$v$r.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['mech_ms'])"
  done
  timeout 300 python bench.py --config cfg3 --steps 20 --warmup 3 > gpurun_out/bench_cfg3_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg3_$v.json').read().strip().splitlines()[-1]); ps=d['config']['per_step']; print('$v cfg3', round(sum(p['ms'] for p in ps),1), [round(p['ms'],1) for p in ps[-5:]])"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
