#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_fullsize.py -q -x -k "frontend or cfg5" > $o/t.log 2>&1; tail -3 $o/t.log
for bm in mine cg; do
  MOE_FRONT_BARRIER=$bm MOE_DECODE_PREFETCH_MB=0 timeout 120 python exp/front_trace.py cfg5 > $o/trace_$bm.txt 2>&1; echo "== $bm"; cat $o/trace_$bm.txt
done
for rep in 1 2; do
  for v in "0 mine" "1 mine" "1 cg"; do
    set -- $v
    MOE_FRONTEND=$1 MOE_FRONT_BARRIER=$2 timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"$1 $2\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
