#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 300 python tools/dbg_row.py > $O/dbg.log 2>&1; echo dbg=$?; cat $O/dbg.log | tail -40
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 --steps 5 > $O/b4.json 2>$O/b4.err && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mech_row -s 3 -c 1 -o $O/prof_row python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 --steps 5 > $O/ncu.log 2>&1; echo ncu=$?
