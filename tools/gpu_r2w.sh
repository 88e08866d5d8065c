#!/bin/bash
# A/B on one box: two-tile units (tile7 depth 2) at 4 vs 5 CTAs per SM (cfg5 on one GPU, onco)
O=gpurun_out/r2w; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_mech.cu /tmp/km_orig.cu
for v in d2m4 d2m5 d2m4 d2m5; do
  cp tools/ab2/km_$v.cu paper_2503_10796_b200/csrc/kernels_mech.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || echo build_$v failed
  timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --strong-steps 0 > $O/cfg5_$v.json 2>$O/cfg5_$v.err || echo cfg5_$v failed
  timeout 600 python bench.py --config onco --steps 20 --warmup 3 --no-cpu-baseline > $O/onco_$v.json 2>$O/onco_$v.err || echo onco_$v failed
  python -c "import json;d=json.load(open('$O/cfg5_$v.json'));e=json.load(open('$O/onco_$v.json'));print('$v cfg5', round(d['ms_per_step'],2), d['roofline'].get('mech_ms'), 'onco', round(e['ms_per_step'],4))"
done
cp /tmp/km_orig.cu paper_2503_10796_b200/csrc/kernels_mech.cu
