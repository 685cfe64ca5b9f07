#!/bin/bash
# fused front end: where the time goes (phase stamps), prefetch inline / side / off, same box
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
for pf in side inline; do
  for mb in 0 64; do
    MOE_FRONT_PREFETCH=$pf MOE_DECODE_PREFETCH_MB=$mb timeout 120 python exp/front_trace.py cfg5 > $o/trace_${pf}_${mb}.txt 2>&1
    echo "== $pf $mb"; cat $o/trace_${pf}_${mb}.txt
  done
done
for rep in 1 2; do
  for v in "0 side 64" "1 side 64" "1 inline 64" "1 side 0"; do
    set -- $v
    MOE_FRONTEND=$1 MOE_FRONT_PREFETCH=$2 MOE_DECODE_PREFETCH_MB=$3 timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"v\": \"$1 $2 $3\", \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
MOE_FRONT_PREFETCH=side timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $o/launches_cfg5_side.csv python bench_configs.py --configs cfg5 --steps 10 --warmup 2 --graphs > /dev/null 2>&1
python exp/ncu_csv.py < $o/launches_cfg5_side.csv 2>/dev/null | head -12
MOE_FRONT_PREFETCH=side timeout 300 ncu --set full --import-source on --clock-control none -k regex:frontend -s 4 -c 1 -o $o/front_full python bench_configs.py --configs cfg5 --steps 5 --warmup 2 > /dev/null 2>&1
ls $o
