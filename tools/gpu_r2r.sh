#!/bin/bash
# SIR (round keys, short wrap), dense kernel contact prefilter; counters-off parity tests
O=gpurun_out/r2r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg4.json 2>$O/cfg4.err; echo cfg4=$?
python -c "import json;d=json.load(open('$O/cfg4.json'));print('cfg4', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/cfg3.json 2>$O/cfg3.err; echo cfg3=$?
python -c "import json;d=json.load(open('$O/cfg3.json'));print('cfg3', round(d['ms_per_step'],2), d['roofline']['t_total_ms'], d['roofline']['frac'])"
timeout 1500 python -m pytest tests/test_gpu_sir.py tests/test_gpu_cfg3.py tests/test_gpu_mech.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
