#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
for rep in 1 2; do
  for v in "0 64" "1 64" "0 0" "1 0"; do
    set -- $v
    MOE_DEBUG_GRAPH_MIN=$1 MOE_DECODE_PREFETCH_MB=$2 timeout 300 python bench_configs.py --configs cfg5 --steps 300 --graphs | sed "s/^{/{\"v\": \"min$1 pf$2\", \"rep\": $rep, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], 'p50', round(d['p50_ms']*1e3,1), 'p99', round(d['p99_ms']*1e3,1), 'mean', round(d['ms_per_step']*1e3,2))"
