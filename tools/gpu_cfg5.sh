#!/bin/bash
# cfg5 (1.7e9 agents) on one GPU after the lean-workspace change, plus the GPU suite.
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/mem.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -c 600 gpurun_out/bench_cfg2.json
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo "cfg5 rc=$?"
tail -c 1500 gpurun_out/bench_cfg5.json; tail -5 gpurun_out/bench_cfg5.err
