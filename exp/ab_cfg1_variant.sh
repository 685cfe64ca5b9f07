#!/bin/bash
# cfg1 (2048 tokens, mean 512 rows per expert): K4 variant A/B, CUDA graphs, 2 alternations
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
for rep in 1 2; do
for v in auto 2sm 1sm swap64; do
  if [ $v = auto ]; then unset MOE_GEMM_VARIANT; else export MOE_GEMM_VARIANT=$v; fi
  timeout 300 python bench_configs.py --configs cfg1 --steps 300 --graphs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1), round(d['k4_tflops']))" >> $o/ab.txt
done
done
unset MOE_GEMM_VARIANT
cat $o/ab.txt
