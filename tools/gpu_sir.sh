#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sir.py -q -x > gpurun_out/pytest_sir.log 2>&1
tail -3 gpurun_out/pytest_sir.log
timeout 300 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg4.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
