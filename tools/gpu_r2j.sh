#!/bin/bash
# full GPU suite with tile7 as the default, smoke, the default bench line (cpu baseline,
# e2e, strong_cfg5 T_1) and the reference arm
O=gpurun_out/r2j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
nproc; lscpu | grep "Model name"; free -g | head -2
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2j/bench_default.json'))
print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'], d.get('step_ms'))
print('cpu', d.get('cpu_baseline'))
print('e2e', {k:d['e2e'][k] for k in ('value','ms_per_step')} if d.get('e2e') else None)
print('strong', d.get('strong_cfg5'))
PY
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
cut -c1-400 $O/bench_reference.json
