#!/bin/bash
# session 3: source-level ncu captures of k_mech_dense (cfg3 step 16, 64M agents) and
# k_sir_update (cfg4), for the stall/source breakdown
O=gpurun_out/s3b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mech_dense -s 16 -c 1 -o $O/prof_dense python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/ncu_dense.log 2>&1; echo dense=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sir_update -s 3 -c 1 -o $O/prof_sir python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sir.log 2>&1; echo sir=$?
ls -la $O
