#!/bin/bash
# decode stack: next-layer L2 prefetch from K4's idle CTAs (MOE_DECODE_PREFETCH_NEXT_MB) — 8-layer graph, cfg5
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
MOE_DECODE_PREFETCH_NEXT_MB=96 timeout 600 python -m pytest tests/test_gpu_graph_stack.py -q -x 2>&1 | tail -1
for rep in 1 2; do
for mb in 0 64 96 128; do
  MOE_DECODE_PREFETCH_NEXT_MB=$mb timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 200 --stack-graph 8 2>/dev/null \
    | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    d=json.loads(l); print('next_mb=$mb', d['config'], round(d['p50_layer_ms']*1e3,1), round(d['p99_layer_ms']*1e3,1))" >> $o/ab.txt
done
done
cat $o/ab.txt
