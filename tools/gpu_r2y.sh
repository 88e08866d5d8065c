#!/bin/bash
# parity subsets on the new grid build (single-pass scan, ILP) + the graph-replay test
O=gpurun_out/r2y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_graph.py tests/test_gpu_mech.py tests/test_gpu_slabs.py tests/test_gpu_sfc.py tests/test_gpu_cfg3.py tests/test_gpu_cfg5_full.py tests/test_gpu_onco.py tests/test_gpu_fuzz.py -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
