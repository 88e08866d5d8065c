#!/bin/bash
# SIR occupancy variants, CUDA-graph line, cfg1 line, ncu launch list + full capture of
# the tile7 mechanics kernel + fp64 SASS op counts
O=gpurun_out/r2k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg4_m4.json 2>$O/cfg4_m4.err; echo cfg4_m4=$?
python -c "import json;d=json.load(open('$O/cfg4_m4.json'));print('m4', d['ms_per_step'], d['roofline']['frac'])"
BDM_NVCC_EXTRA=-DBDM_SIR_MINB=3 python -c "import __graft_entry__ as g; g.build()" > $O/build3.log 2>&1
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg4_m3.json 2>$O/cfg4_m3.err; echo cfg4_m3=$?
python -c "import json;d=json.load(open('$O/cfg4_m3.json'));print('m3', d['ms_per_step'], d['roofline']['frac'])"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 > $O/graph.json 2>$O/graph.err; echo graph=$?
python -c "import json;d=json.load(open('$O/graph.json'));print('plain', d['ms_per_step'], 'graph', d.get('graph'))"
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-e2e --strong-steps 0 > $O/cfg1.json 2>$O/cfg1.err; echo cfg1=$?
cut -c1-300 $O/cfg1.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/plain_ll.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_ll.log 2>&1; echo ll=$?
timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 --csv --log-file $O/fp64_counts.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_fp64.log 2>&1; echo fp64=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_mech python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_full.log 2>&1; echo full=$?
