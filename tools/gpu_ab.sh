#!/bin/bash
# A/B of the phase-1 walk (BDM_WALK_LAZY) + the in-place keep-order e2e path.
mkdir -p gpurun_out
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sfc.py -q -x > gpurun_out/pytest_sfc.log 2>&1; tail -2 gpurun_out/pytest_sfc.log
for r in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_A$r.json 2> gpurun_out/bench_A.err
python -c "import json; d=json.loads(open('gpurun_out/bench_A$r.json').read().strip().splitlines()[-1]); print('A', d['ms_per_step'], d['roofline']['mech_ms'], d['e2e']['ms_per_step'])"
done
BDM_NVCC_EXTRA="-DBDM_WALK_LAZY" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/buildB.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mech.py -q -x -k "tile and not tile_v1 and not tile_4cta" > gpurun_out/pytest_B.log 2>&1; tail -2 gpurun_out/pytest_B.log
for r in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_B$r.json 2> gpurun_out/bench_B.err
python -c "import json; d=json.loads(open('gpurun_out/bench_B$r.json').read().strip().splitlines()[-1]); print('B', d['ms_per_step'], d['roofline']['mech_ms'])"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
