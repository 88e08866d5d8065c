timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_cfg3.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_d1.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_d1.log
timeout 600 python bench.py --config cfg3 --steps 16 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_d1.log 2>&1; echo cfg3=$?
tail -1 gpurun_out/bench_cfg3_d1.log | cut -c1-1500
