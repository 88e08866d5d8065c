#!/bin/bash
# A/B of kernels_mech variants (tools/variants/*.cu): bench + one ncu full capture each
O=gpurun_out/r2o; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_mech.cu /tmp/km_orig.cu
for v in v1 v2; do
  cp tools/variants/kernels_mech_$v.cu paper_2503_10796_b200/csrc/kernels_mech.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1; echo build_$v=$?
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 --steps 20 > $O/bench_$v.json 2>$O/bench_$v.err; echo bench_$v=$?
  python -c "import json;d=json.load(open('$O/bench_$v.json'));r=d['roofline'];print('$v', d['ms_per_step'], d['value'], r['achieved'], r['frac'])"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_tile6 -s 5 -c 1 -o $O/prof_$v python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --strong-steps 0 --no-graph > $O/ncu_$v.log 2>&1; echo full_$v=$?
done
cp /tmp/km_orig.cu paper_2503_10796_b200/csrc/kernels_mech.cu
