#!/bin/bash
# One GPU iteration: parity tests, a short bench, and an ncu capture of the tile kernel.
# usage (under gpurun): bash tools/gpu_cycle.sh TAG [extra bench args]
TAG=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_$TAG.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]); r=d['roofline']; print('value %.3g ms_step %.3f mech %.3f grid %.3f frac %.3f' % (d['value'], d['ms_per_step'], r['mech_ms'], r['grid_ms'], r['frac']))"
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mech -s 4 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
