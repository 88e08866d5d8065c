#!/bin/bash
# tile-kernel restructure: parity subsets + cfg2/cfg5 benches
O=gpurun_out/s2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_mech.py tests/test_gpu_sfc.py tests/test_gpu_fuzz.py tests/test_gpu_graph.py tests/test_gpu_onco.py tests/test_gpu_slabs.py -q -x -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
for r in 1 2; do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/bench_$r.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/bench_$r.json').read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step'],4), round(d['roofline']['mech_ms'],4), round(d['roofline']['grid_ms'],4))"
done
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg5.json 2>/dev/null
python -c "import json; d=json.loads(open('$O/bench_cfg5.json').read().strip().splitlines()[-1]); print('cfg5', round(d['ms_per_step'],2))"
timeout 900 python -m pytest tests/test_gpu_cfg5_full.py tests/test_gpu_cfg3.py -q -x -m gpu > $O/pytest2.log 2>&1; echo pytest2=$?; tail -3 $O/pytest2.log
