#!/bin/bash
# Parity tests, then a short bench per mechanics kernel, then ncu of the first one.
# usage (under gpurun): bash tools/gpu_multi.sh TAG "k1 k2 ..." [pytest-args]
TAG=$1; KS=$2; shift 2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_$TAG.log
for k in $KS; do
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mech-kernel $k > gpurun_out/bench_${TAG}_k$k.log 2>&1; echo bench k$k=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_${TAG}_k$k.log').read().strip().splitlines()[-1]); r=d['roofline']; print('k$k value %.3g ms_step %.3f mech %.3f grid %.3f frac %.3f' % (d['value'], d['ms_per_step'], r['mech_ms'], r['grid_ms'], r['frac']))"
done
K0=${KS%% *}
ncu --set full --clock-control none --import-source on -k regex:k_mech -s 4 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mech-kernel $K0 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
