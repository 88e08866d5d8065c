#!/bin/bash
# Round-end refresh of every committed measurement: GPU suite, smoke, the default bench
# line (N=1, cfg2) and the reference arm, the other configs, the launch list and one
# ncu --set full capture of the dominant kernel.
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
for c in cfg3 cfg4 soma onco aura; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?
done
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_ll.log 2>&1; echo ll=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 2 -c 1 -o $O/prof_mech python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1; echo full=$?
