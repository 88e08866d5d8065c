#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_all.log)"
timeout 600 python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_auto.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg5_auto.json').read().strip().splitlines()[-1]); print('cfg5 auto', round(d['ms_per_step'],2), round(d['roofline']['mech_ms'],2))"
for r in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2_auto.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_auto.json').read().strip().splitlines()[-1]); print('cfg2 auto', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4))"
done
timeout 300 python bench.py --config onco --steps 20 --warmup 3 > gpurun_out/bench_onco.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_onco.json').read().strip().splitlines()[-1]); print('onco', d['ms_per_step'])"
timeout 300 python bench.py --config cfg3 --steps 20 --warmup 3 > gpurun_out/bench_cfg3.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_cfg3.json').read().strip().splitlines()[-1]); print('cfg3', sum(p['ms'] for p in d['config']['per_step']))"
