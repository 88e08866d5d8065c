#!/bin/bash
# toroidal mechanics parity; depth-2 tile7 at 5 CTAs/SM; regression subsets
O=gpurun_out/r2z; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_torus.py -q -m gpu > $O/pytest_torus.log 2>&1; echo torus=$?; tail -15 $O/pytest_torus.log
timeout 2000 python -m pytest tests/test_gpu_mech.py tests/test_gpu_cfg5_full.py tests/test_gpu_onco.py tests/test_gpu_fuzz.py tests/test_gpu_graph.py tests/test_gpu_sfc.py tests/test_gpu_slabs.py tests/test_gpu_sir.py -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
