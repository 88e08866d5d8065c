#!/bin/bash
# session 4: tile7 with 8-warp two-tile units (tile_depth 3) against the default (depth 1)
# at cfg2: tile parity tests, then two bench lines per depth
O=gpurun_out/s4d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_mech.py -m gpu -q -x -p no:cacheprovider -k "tile7" > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
for d in 1 3 1 3; do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --tile-depth $d > $O/bench_d$d.json 2> $O/bench_d$d.err
  python -c "import json; d=json.loads(open('$O/bench_d$d.json').read().strip().splitlines()[-1]); print('depth $d', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
done
