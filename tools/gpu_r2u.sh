#!/bin/bash
# A/B on one box: grid build with one agent per thread vs kGridIlp = 4 (k_key, k_scatter)
O=gpurun_out/r2u; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_grid.cu /tmp/kg_orig.cu
for v in old ilp old ilp; do
  cp tools/ab/kg_$v.cu paper_2503_10796_b200/csrc/kernels_grid.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || echo build_$v failed
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 --steps 30 > $O/bench_$v.json 2>$O/bench_$v.err || echo bench_$v failed
  python -c "import json;d=json.load(open('$O/bench_$v.json'));r=d['roofline'];print('$v', round(d['ms_per_step'],4), 'mech', round(r['mech_ms'],4), 'grid', round(r['grid_ms'],4))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_key|k_scatter|k_fix_gather|k_scan|k_zero" -c 40 --csv --log-file $O/grid_ilp.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu.log 2>&1; echo ncu=$?
cp /tmp/kg_orig.cu paper_2503_10796_b200/csrc/kernels_grid.cu
python -c "import __graft_entry__ as g; g.build()" > $O/build_final.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_slabs.py tests/test_gpu_sfc.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
