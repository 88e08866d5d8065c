#!/bin/bash
# full GPU suite, smoke, default bench line, reference arm, ncu launch list and full
# captures of the mechanics (tile7, 6 CTAs) and SIR kernels
O=gpurun_out/r2t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2t/bench_default.json'))
print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'], d['roofline']['frac'], d.get('step_ms'))
print('graph', d.get('graph'))
print('cpu', d.get('cpu_baseline',{}).get('value'))
print('e2e', {k:d['e2e'][k] for k in ('value','ms_per_step')} if d.get('e2e') else None)
s=d.get('strong_cfg5') or {}; print('strong', s.get('ms_per_step'), s.get('exchange_ms'))
PY
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
cut -c1-300 $O/bench_reference.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/plain_ll.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_ll.log 2>&1; echo ll=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_mech python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_full.log 2>&1; echo full=$?
timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 --csv --log-file $O/fp64_counts.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_fp64.log 2>&1; echo fp64=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sir_update -s 3 -c 1 -o $O/prof_sir python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sir.log 2>&1; echo sir=$?
