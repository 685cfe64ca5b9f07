#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
for rep in 1 2; do
  for v in 1sm 2sm; do
    MOE_GEMM_VARIANT=$v timeout 600 python bench_configs.py --configs cfg3,cfg1 --steps 200 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], round(d['tokens_per_s']), round(d['p50_ms'],3), round(d['p99_ms'],3), d['phase_ms_median']['gemm1_ms'], d['phase_ms_median']['gemm2_ms'])"
