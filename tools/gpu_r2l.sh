#!/bin/bash
# the other config lines with the default kernel, and the graph measurement
O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 300 python tools/dbg_graph.py > $O/dbg_graph.log 2>&1; echo dbg_graph=$?; cat $O/dbg_graph.log | tail -4
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
python -c "import json;d=json.load(open('$O/bench_cfg3.json'));print('cfg3', d['ms_per_step'], d['value'], d['roofline'], d.get('cpu_baseline',{}).get('value'))"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --strong-steps 0 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
python -c "import json;d=json.load(open('$O/bench_cfg5.json'));print('cfg5', d['ms_per_step'], d['value'], d['roofline'].get('mech_ms'), d.get('cpu_baseline',{}).get('value'))"
timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
python -c "import json;d=json.load(open('$O/bench_cfg4.json'));print('cfg4', d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline'))"
for c in onco soma aura; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --strong-steps 0 > $O/graph.json 2>$O/graph.err; echo graph=$?
python -c "import json;d=json.load(open('$O/graph.json'));print('plain', d['ms_per_step'], 'graph', d.get('graph'))"
timeout 600 python bench.py --force-slabs --no-cpu-baseline --strong-steps 0 --steps 20 > $O/slabs1.json 2>$O/slabs1.err; echo slabs1=$?
cut -c1-600 $O/slabs1.json
