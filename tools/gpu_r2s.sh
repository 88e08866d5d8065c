#!/bin/bash
# A/B on one box: dense kernel with / without the contact prefilter (cfg3, 20 steps)
O=gpurun_out/r2s; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_mech.cu /tmp/km_orig.cu
for v in dense_off dense_on dense_off dense_on; do
  cp tools/ab/km_$v.cu paper_2503_10796_b200/csrc/kernels_mech.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || echo build_$v failed
  timeout 900 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg3_$v.json 2>$O/cfg3_$v.err || echo cfg3_$v failed
  python -c "import json;d=json.load(open('$O/cfg3_$v.json'));p=d['config']['per_step'];print('$v', round(d['roofline']['t_total_ms'],1), [round(x['ms'],1) for x in p[-4:]])"
done
cp /tmp/km_orig.cu paper_2503_10796_b200/csrc/kernels_mech.cu
