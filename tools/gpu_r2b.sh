#!/bin/bash
# row kernel: mech parity (row param) + fuzz + bench A/B
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mech.py -q -x -p no:cacheprovider -k "row" > $O/pytest_row.log 2>&1; echo pytest_row=$?; tail -15 $O/pytest_row.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > $O/pytest_fuzz.log 2>&1; echo fuzz=$?; tail -15 $O/pytest_fuzz.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 > $O/bench_row.json 2> $O/bench_row.err; echo bench_row=$?
python -c "import json;d=json.load(open('$O/bench_row.json'));print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'])"
tail -3 $O/bench_row.err
