#!/bin/bash
# combine launched programmatically behind K4 (MOE_PDL_FRONT bit 2 eager / bit 8 graphs) at decode
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
MOE_PDL_FRONT=15 timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_graph_stack.py tests/test_gpu_layer.py -q -x 2>&1 | tail -1
for rep in 1 2; do
for m in 1 15; do
  MOE_PDL_FRONT=$m timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m graph', d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))" >> $o/ab.txt
  MOE_PDL_FRONT=$m timeout 300 python bench_configs.py --configs cfg5 --steps 200 --stack-graph 8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m stack8', d['config'], round(d['p50_layer_ms']*1e3,1), round(d['p99_layer_ms']*1e3,1))" >> $o/ab.txt
  MOE_PDL_FRONT=$m timeout 300 python bench_configs.py --configs cfg5 --steps 300 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m eager', d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))" >> $o/ab.txt
done
done
cat $o/ab.txt
