#!/bin/bash
# A/B: 128-token swap-AB tiles (fused GEMM1+GEMM2) vs the 1-SM kernel on cfg1 / cfg3 / cfg2
out=gpurun_out/ab_swap128.jsonl
: > $out
for rep in 1 2; do
  for v in 1sm swap128; do
    export MOE_GEMM_VARIANT=$v
    timeout 300 python bench_configs.py --configs cfg1,cfg3 --steps 200 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg1 --steps 200 --graphs | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
  done
done
for v in 1sm swap128; do
  MOE_GEMM_VARIANT=$v timeout 300 python bench.py --steps 100 --warmup 10 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_swap128_cfg2.jsonl
done
