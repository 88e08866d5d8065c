#!/bin/bash
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 300 python tools/dbg_row3.py > $O/dbg3.log 2>&1; echo dbg=$?; head -60 $O/dbg3.log
