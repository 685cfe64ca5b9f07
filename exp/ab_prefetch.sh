#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 300 python -m pytest tests/test_gpu_gemm_variants.py tests/test_gpu_layer.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for rep in 1 2; do
  for mb in 0 32 64 96; do
    MOE_DECODE_PREFETCH_MB=$mb timeout 300 python bench_configs.py --configs cfg5,cfg5s12 --steps 300 --graphs | sed "s/^{/{\"mb\": $mb, \"rep\": $rep, \"graphs\": 1, /" >> $o/cfg.jsonl
    MOE_DECODE_PREFETCH_MB=$mb timeout 300 python bench_configs.py --configs cfg5 --steps 300 | sed "s/^{/{\"mb\": $mb, \"rep\": $rep, \"graphs\": 0, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['mb'], d['rep'], d['graphs'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
