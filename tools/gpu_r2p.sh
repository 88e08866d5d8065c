#!/bin/bash
# A/B of kernels_mech variants v1 (6 CTAs) / v3 (+ tile drawn one ahead) / v4 (+ contact-reach trimming)
O=gpurun_out/r2p; mkdir -p $O
cp paper_2503_10796_b200/csrc/kernels_mech.cu /tmp/km_orig.cu
for v in v1 v3 v4 v1 v3 v4; do
  cp tools/variants/kernels_mech_$v.cu paper_2503_10796_b200/csrc/kernels_mech.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || echo build_$v failed
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 --steps 30 > $O/bench_$v.json 2>$O/bench_$v.err || echo bench_$v failed
  python -c "import json;d=json.load(open('$O/bench_$v.json'));r=d['roofline'];print('$v', round(d['ms_per_step'],4), 'mech', round(r['mech_ms'],4), 'grid', round(r['grid_ms'],4), r['work_per_launch']['cand'])"
done
cp tools/variants/kernels_mech_v4.cu paper_2503_10796_b200/csrc/kernels_mech.cu
python -c "import __graft_entry__ as g; g.build()" > $O/build_final.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_fuzz.py tests/test_gpu_sfc.py tests/test_gpu_slabs.py -x -q -m gpu > $O/pytest_v4.log 2>&1; echo pytest_v4=$?; tail -2 $O/pytest_v4.log
cp /tmp/km_orig.cu paper_2503_10796_b200/csrc/kernels_mech.cu
