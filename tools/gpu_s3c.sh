#!/bin/bash
# session 3 A/B of the dense kernel: variants given as BDM_NVCC_EXTRA strings; per
# variant the dense/cfg3 parity tests and the cfg3 bench (20 steps)
O=gpurun_out/s3c; mkdir -p $O
i=0
for X in "$@"; do
  i=$((i+1))
  BDM_NVCC_EXTRA="$X" python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build_v$i.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_cfg3.py tests/test_gpu_mech.py -m gpu -q -x -k "dense or cfg3" -p no:cacheprovider > $O/pytest_v$i.log 2>&1
  echo "v$i [$X] tests: $(tail -1 $O/pytest_v$i.log)"
  timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_v$i.json 2> $O/bench_cfg3_v$i.err
  python -c "import json; d=json.loads(open('$O/bench_cfg3_v$i.json').read().strip().splitlines()[-1]); print('v$i', round(d['ms_per_step']*20,1), [round(s['ms'],1) for s in d['config']['per_step'][-4:]])"
done
python -c "from paper_2503_10796_b200 import build; build.build(force=True)" > $O/build.log 2>&1
