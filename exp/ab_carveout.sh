#!/bin/bash
# decode: prefetch / front end with the K4 carveout, prefetch size sweep (graph traces + bench)
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
for mb in 0 64 96 128; do
  TRACE_GRAPHS=1 MOE_DECODE_PREFETCH_MB=$mb timeout 120 python exp/front_trace.py cfg5 2>&1 | tail -1 | sed "s/^/pf$mb /"
done
for rep in 1 2; do
  for mb in 0 64 96 128; do
    MOE_DECODE_PREFETCH_MB=$mb timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"pf$mb\", \"rep\": $rep, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], 'p50', round(d['p50_ms']*1e3,1), 'p99', round(d['p99_ms']*1e3,1), 'mean', round(d['ms_per_step']*1e3,2))"
