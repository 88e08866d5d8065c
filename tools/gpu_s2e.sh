#!/bin/bash
# SIR after the warp-cooperative search: parity, cfg4 line, ncu full capture
O=gpurun_out/s2e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_sir.py -q -m gpu > $O/pytest_sir.log 2>&1; echo pytest=$?; tail -1 $O/pytest_sir.log
timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
python -c "import json;d=json.load(open('$O/bench_cfg4.json'));print('cfg4', d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sir_update -s 3 -c 1 -o $O/prof_sir python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sir.log 2>&1; echo sir=$?
