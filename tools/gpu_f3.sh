#!/bin/bash
# Row f3: aura codec parity, memcheck, and the cfg2 slab-aura measurement.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_aura.py -x -q > gpurun_out/pytest_aura.log 2>&1
tail -15 gpurun_out/pytest_aura.log


timeout 600 python bench.py --config aura --steps 5 --warmup 3 > gpurun_out/bench_aura.json 2> gpurun_out/bench_aura.err
echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_aura.json; tail -3 gpurun_out/bench_aura.err
