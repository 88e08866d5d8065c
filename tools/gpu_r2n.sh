#!/bin/bash
# tile7 with balanced walk pieces
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_fuzz.py tests/test_gpu_sfc.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 --steps 20 > $O/bench.json 2>$O/bench.err; echo bench=$?
python -c "import json;d=json.load(open('$O/bench.json'));r=d['roofline'];print('bench', d['ms_per_step'], d['value'], r.get('kernel_ms'), r['achieved'], r['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 --csv --log-file $O/occ.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_occ.log 2>&1; echo occ=$?
cat $O/occ.csv | cut -c1-300 | tail -6
