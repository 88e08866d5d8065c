#!/bin/bash
# SIR: infected_fine inlined (no stack copy of the arguments); register budget A/B
O=gpurun_out/r2q; mkdir -p $O
for mb in 4 3 2 4 3; do
  BDM_NVCC_EXTRA=-DBDM_SIR_MINB=$mb python -c "import __graft_entry__ as g; g.build()" > $O/build_$mb.log 2>&1 || echo build_$mb failed
  timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg4_$mb.json 2>$O/cfg4_$mb.err || echo cfg4_$mb failed
  python -c "import json;d=json.load(open('$O/cfg4_$mb.json'));print('minB $mb', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
done
python -c "import __graft_entry__ as g; g.build()" > $O/build_final.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sir.py -x -q -m gpu > $O/pytest_sir.log 2>&1; echo pytest_sir=$?; tail -2 $O/pytest_sir.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sir_update -s 3 -c 1 -o $O/prof_sir python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sir.log 2>&1; echo ncu=$?
