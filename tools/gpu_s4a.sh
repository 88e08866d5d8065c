#!/bin/bash
# session-4 (final) refresh of the committed measurements: GPU suite, smoke, the default bench
# line and the reference arm, every other config line, the launch list, ncu full
# captures of the mechanics and SIR kernels, fp64 SASS counts of the mechanics kernel
O=gpurun_out/s4a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
timeout 300 python bench.py --config cfg1 --steps 100 --warmup 5 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo cfg1=$?
timeout 1200 python bench.py --config cfg3 --steps 20 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --strong-steps 0 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
for c in onco soma aura; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?
done
timeout 600 python bench.py --force-slabs --no-cpu-baseline --strong-steps 0 --steps 20 > $O/bench_slabs1.json 2>$O/bench_slabs1.err; echo slabs1=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/plain_ll.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_ll.log 2>&1; echo ll=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_mech python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_full.log 2>&1; echo full=$?
timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 --csv --log-file $O/fp64_counts.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_fp64.log 2>&1; echo fp64=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sir_update -s 3 -c 1 -o $O/prof_sir python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sir.log 2>&1; echo sir=$?
