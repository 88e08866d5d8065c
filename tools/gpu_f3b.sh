#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_aura.py -q > gpurun_out/pytest_aura.log 2>&1
tail -3 gpurun_out/pytest_aura.log
timeout 300 python bench.py --config aura --steps 5 --warmup 3 > gpurun_out/bench_aura.json 2> gpurun_out/bench_aura.err
python -c "import json; d=json.loads(open('gpurun_out/bench_aura.json').read().strip().splitlines()[-1]); print(d['config']['ratio_raw_over_stream'], [(r['encode_ms'], r['decode_ms']) for r in d['config']['per_step']])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_aura.csv python bench.py --config aura --steps 2 --warmup 3 > gpurun_out/ncu_aura.log 2>&1
grep -E "k_lz4|k_aura" gpurun_out/launches_aura.csv | awk -F'","' '{print $5" "$NF}' | sed 's/(.*) / /' | cut -c1-80
