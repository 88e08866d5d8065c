#!/bin/bash
# Row f1: parity of the sorting-frequency / Hilbert options, the whole GPU suite, and
# the cfg2 sweep (tile order x sort frequency x start order).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sfc.py -x -q > gpurun_out/pytest_sfc.log 2>&1
tail -3 gpurun_out/pytest_sfc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/f1_sweep.jsonl
for spec in "0 1" "1 1" "0 1 --shuffle" "0 0" "0 0 --shuffle" "1 0 --shuffle" "0 10 --shuffle" "0 10" ; do
  set -- $spec
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline \
      --tile-order $1 --sort-every $2 $3 >> gpurun_out/f1_sweep.jsonl 2>> gpurun_out/f1_sweep.err
  echo "spec $spec rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/f1_sweep.jsonl"):
    d = json.loads(l)
    print(d.get("f1"), round(d["ms_per_step"], 3), d["roofline"]["mech_ms"], d["roofline"]["grid_ms"])
PY
