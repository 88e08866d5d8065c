#!/bin/bash
# session 4: HEAD health check (full GPU suite, smoke, default bench line, cfg5 with depth 2/auto)
O=gpurun_out/${BDM_OUT:-s4g}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --strong-steps 0 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
