#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py -q -x > $o/t.log 2>&1; tail -3 $o/t.log
MOE_DECODE_PREFETCH_MB=0 timeout 120 python exp/front_trace.py cfg5 > $o/trace0.txt 2>&1; cat $o/trace0.txt
timeout 120 python exp/front_trace.py cfg5 > $o/trace64.txt 2>&1; cat $o/trace64.txt
for rep in 1 2; do
  for fe in 0 1; do
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"$fe\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg5 --steps 300 | sed "s/^{/{\"v\": \"$fe\", \"rep\": $rep, \"graphs\": 0, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
