#!/bin/bash
# decode weight warm-up during the fused front end: first-wave tile boxes vs linear bulk vs side stream
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 300 python -m pytest tests/test_gpu_frontend.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for rep in 1 2; do
  for v in "tiles 64" "linear 64" "side 64" "tiles 0" "tiles 32" "tiles 96" "tiles 128"; do
    set -- $v
    MOE_FRONT_PREFETCH=$1 MOE_DECODE_PREFETCH_MB=$2 timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"$1 $2\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], 'p50', round(d['p50_ms']*1e3,1), 'p99', round(d['p99_ms']*1e3,1), 'mean', round(d['ms_per_step']*1e3,2), 'k4', round(d['phase_ms_median']['gemm1_ms']*1e3,1))"
for mb in 0 64; do MOE_DECODE_PREFETCH_MB=$mb timeout 120 python exp/front_trace.py cfg5 > $o/trace$mb.txt 2>&1; cat $o/trace$mb.txt; done
