#!/bin/bash
# Full GPU suite (incl. the cfg5 full-size sampled parity), default bench, aura launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['mech_ms'], d['roofline']['grid_ms'])"


timeout 300 python bench.py --config aura --steps 3 --warmup 3 > gpurun_out/bench_aura.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_aura.json').read().strip().splitlines()[-1]); print([(r['encode_ms'], r['decode_ms']) for r in d['config']['per_step']])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lz4 -c 2 -o gpurun_out/prof_lz4 python bench.py --config aura --steps 1 --warmup 3 > gpurun_out/ncu_lz4.log 2>&1
echo "ncu rc=$?"
