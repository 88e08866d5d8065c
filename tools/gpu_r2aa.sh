#!/bin/bash
# toroidal parity (bdm_step path), bdm_run_host parity, default bench line with the pipelined e2e
O=gpurun_out/r2aa; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_torus.py tests/test_gpu_e2e.py -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -15 $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline --strong-steps 0 > $O/bench.json 2>$O/bench.err; echo bench=$?
python -c "import json;d=json.load(open('$O/bench.json'));print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'], json.dumps(d['e2e']))"
