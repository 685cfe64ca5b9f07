#!/bin/bash
# fused decode front end (MOE_FRONTEND=1) vs gate / finish / dispatch launches, same box
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 400 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_fullsize.py -k "frontend or cfg5" -q -x > $o/t.log 2>&1; tail -3 $o/t.log
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
MOE_FRONTEND=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $o/launches_cfg5.csv python bench_configs.py --configs cfg5 --steps 10 --warmup 2 --graphs > /dev/null 2>&1
python exp/ncu_csv.py < $o/launches_cfg5.csv 2>/dev/null | head -40
