#!/bin/bash
# session-2 baseline: build, mech parity subset, default bench, ncu full capture of k_mech
O=gpurun_out/s2a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mech.py -q -m gpu -x > $O/pytest_mech.log 2>&1; echo pytest=$?; tail -3 $O/pytest_mech.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/s2a/bench_default.json'))
print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'], d['roofline']['frac'], d.get('step_ms'))
print('graph', d.get('graph'))
print('e2e', {k:d['e2e'][k] for k in ('value','ms_per_step') if k in d['e2e']} if d.get('e2e') else None)
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_mech python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_full.log 2>&1; echo full=$?
