#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
timeout 900 python -m pytest tests -m gpu -q -x > $o/t.log 2>&1; tail -3 $o/t.log
for st in 0 1; do
  MOE_GATE_STREAM=$st timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_ -s 3 -c 3 --csv \
    python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg2 stream=$st" >> $o/ab.txt
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg5.csv \
  python bench_configs.py --configs cfg5 --steps 5 --warmup 2 --graphs > /dev/null 2>&1
for rep in 1 2; do
  for fp in 0 1; do
    MOE_FUSE_PLAN=$fp timeout 300 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs | sed "s/^{/{\"fuse_plan\": $fp, \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
    MOE_FUSE_PLAN=$fp timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"fuse_plan\": $fp, \"rep\": $rep, \"graphs\": 0, /" >> $o/cfg.jsonl
  done
done
cat $o/ab.txt
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['fuse_plan'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
