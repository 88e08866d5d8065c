#!/bin/bash
# A/B on one box: grid build ilp (committed) / + single-pass slot scan / + fix_gather 2 per thread;
# then the x-slab line at N = 1 with the new per-rank e2e
O=gpurun_out/r2v; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_grid.cu /tmp/kg_orig.cu
for v in ilp single single_fix2 ilp single single_fix2; do
  cp tools/ab/kg_$v.cu paper_2503_10796_b200/csrc/kernels_grid.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || echo build_$v failed
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 --steps 30 > $O/bench_$v.json 2>$O/bench_$v.err || echo bench_$v failed
  python -c "import json;d=json.load(open('$O/bench_$v.json'));r=d['roofline'];print('$v', round(d['ms_per_step'],4), 'mech', round(r['mech_ms'],4), 'grid', round(r['grid_ms'],4))"
done
cp /tmp/kg_orig.cu paper_2503_10796_b200/csrc/kernels_grid.cu
python -c "import __graft_entry__ as g; g.build()" > $O/build_final.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mech.py tests/test_gpu_slabs.py tests/test_gpu_sfc.py tests/test_gpu_cfg3.py tests/test_gpu_cfg5_full.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 600 python bench.py --force-slabs --no-cpu-baseline --strong-steps 0 --steps 20 > $O/slabs1.json 2>$O/slabs1.err; echo slabs1=$?
python -c "import json;d=json.load(open('$O/slabs1.json'));print('slabs1', d['ms_per_step'], d.get('e2e'))"
