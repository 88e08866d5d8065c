#!/bin/bash
# session-3 health check of HEAD: GPU suite, smoke, default bench, cfg3, cfg4
O=gpurun_out/s3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
for f in default cfg3 cfg4; do python -c "import json,sys; d=json.loads(open('$O/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d.get('roofline',{}).get('mech_ms'), d.get('roofline',{}).get('grid_ms'))"; done
