#!/bin/bash
# full GPU suite, smoke, default bench, ncu full capture of the tile7 kernel
O=gpurun_out/s2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/s2c/bench_default.json'))
print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'], d['roofline']['frac'], d.get('step_ms',{}).get('median'))
print('graph', d.get('graph',{}).get('ms_per_step'), 'e2e', d.get('e2e',{}).get('ms_per_step'), 'cpu', d.get('cpu_baseline',{}).get('value'))
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_mech python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_full.log 2>&1; echo full=$?
