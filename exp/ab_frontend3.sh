#!/bin/bash
# fused front end after the redux top-k / 64-bit barrier / vector id histogram
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_predictor.py -q -x > $o/t.log 2>&1; tail -3 $o/t.log
MOE_DECODE_PREFETCH_MB=64 timeout 120 python exp/front_trace.py cfg5 > $o/trace.txt 2>&1; cat $o/trace.txt
MOE_DECODE_PREFETCH_MB=0 timeout 120 python exp/front_trace.py cfg5 > $o/trace0.txt 2>&1; cat $o/trace0.txt
for rep in 1 2; do
  for fe in 0 1; do
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs | sed "s/^{/{\"fe\": $fe, \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg5 --steps 300 | sed "s/^{/{\"fe\": $fe, \"rep\": $rep, \"graphs\": 0, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['fe'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $o/launches_cfg5.csv python bench_configs.py --configs cfg5 --steps 10 --warmup 2 --graphs > /dev/null 2>&1
python exp/ncu_csv.py < $o/launches_cfg5.csv 2>/dev/null | head -9
