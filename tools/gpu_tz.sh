#!/bin/bash
# tile_depth 2: parity (all mech tests run with the tile_depth2 fixture) and cfg5/cfg2 timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mech.py -q -x > gpurun_out/pytest_tz.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_tz.log)"
for d in 1 2; do
  timeout 600 python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline --tile-depth $d > gpurun_out/bench_cfg5_tz$d.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg5_tz$d.json').read().strip().splitlines()[-1]); print('cfg5 tz$d', round(d['ms_per_step'],2), round(d['roofline']['mech_ms'],2))"
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --tile-depth $d > gpurun_out/bench_cfg2_tz$d.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_tz$d.json').read().strip().splitlines()[-1]); print('cfg2 tz$d', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4))"
done
timeout 300 python bench.py --config onco --steps 20 --warmup 3 > gpurun_out/bench_onco.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_onco.json').read().strip().splitlines()[-1]); print('onco', d['ms_per_step'])"
