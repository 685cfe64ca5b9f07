#!/bin/bash
# where the decode layer's time goes beyond K4: skip-combine timing, prefetch sweep (same box)
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
for rep in 1 2; do
  for v in "64 0" "64 1" "0 0" "32 0" "96 0" "128 0"; do
    set -- $v
    MOE_DECODE_PREFETCH_MB=$1 MOE_DEBUG_SKIP_COMBINE=$2 timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"pf$1 skipc$2\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1), round(d['phase_ms_median']['gemm1_ms']*1e3,1))"
