#!/bin/bash
# combine fused into the swap-AB GEMM2 (MOE_SWAP_COMBINE) at decode
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
true
for rep in 1 2; do
for m in 0 1; do
  MOE_SWAP_COMBINE=$m timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m graph', d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))" >> $o/ab.txt
  MOE_SWAP_COMBINE=$m timeout 300 python bench_configs.py --configs cfg5 --steps 200 --stack-graph 8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m stack8', d['config'], round(d['p50_layer_ms']*1e3,1), round(d['p99_layer_ms']*1e3,1))" >> $o/ab.txt
  MOE_SWAP_COMBINE=$m timeout 300 python bench_configs.py --configs cfg5 --steps 300 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('mask=$m eager', d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))" >> $o/ab.txt
done
done
cat $o/ab.txt
