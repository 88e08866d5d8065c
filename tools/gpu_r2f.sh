#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 300 python tools/dbg_row.py > $O/dbg.log 2>&1; echo dbg=$?; grep "bad fields" $O/dbg.log | grep "kernel 4"
timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider -k "row or fuzz" > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 > $O/b4.json 2>$O/b4.err; echo b4=$?
python -c "import json;d=json.load(open('$O/b4.json'));print('row6', d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'])"



python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 --steps 5 > $O/b4s.json 2>$O/b4s.err && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mech_row -s 5 -c 1 -o $O/prof_row python bench.py --no-cpu-baseline --no-e2e --mech-kernel 4 --steps 5 > $O/ncu.log 2>&1; echo ncu=$?
