#!/bin/bash
# swap-AB GEMM2 in 128-row weight tiles vs 256 (decode tail)
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
timeout 600 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_fullsize.py tests/test_gpu_gemm_variants.py tests/test_gpu_layer.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
MOE_SWAP_HALF2=0 timeout 300 python -m pytest tests/test_gpu_gemm_variants.py tests/test_gpu_layer.py -q -x 2>&1 | tail -1
for h in 0 1; do MOE_SWAP_HALF2=$h TRACE_GRAPHS=1 timeout 120 python exp/front_trace.py cfg5 2>&1 | tail -1 | sed "s/^/half$h /"; done
for rep in 1 2; do
  for h in 0 1; do
    MOE_SWAP_HALF2=$h timeout 300 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs | sed "s/^{/{\"v\": \"half$h\", \"rep\": $rep, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], 'p50', round(d['p50_ms']*1e3,1), 'p99', round(d['p99_ms']*1e3,1), 'mean', round(d['ms_per_step']*1e3,2))"
