#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mech.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider -k "tile7 or tile or fuzz" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for k in 0 5; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mech-kernel $k > $O/b$k.json 2>$O/b$k.err; echo b$k=$?
python -c "import json;d=json.load(open('$O/b$k.json'));print('k$k', d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'])"
done
