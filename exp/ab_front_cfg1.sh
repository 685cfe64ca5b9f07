#!/bin/bash
# fused front end extended to 148 token blocks (cfg1: 64 blocks x 2 K splits) vs the launch chain
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for rep in 1 2; do
  for fe in 0 1; do
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg1,cfg5 --steps 300 --graphs | sed "s/^{/{\"v\": \"fe$fe\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
    MOE_FRONTEND=$fe timeout 300 python bench_configs.py --configs cfg1 --steps 300 | sed "s/^{/{\"v\": \"fe$fe\", \"rep\": $rep, \"graphs\": 0, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['graphs'], d['config'], 'p50', round(d['p50_ms']*1e3,1), 'p99', round(d['p99_ms']*1e3,1), 'mean', round(d['ms_per_step']*1e3,2))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $o/launches_cfg1.csv python bench_configs.py --configs cfg1 --steps 5 --warmup 2 --graphs > /dev/null 2>&1
python exp/ncu_csv.py < $o/launches_cfg1.csv | head -8
