#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?; tail -30 $O/pytest.log
