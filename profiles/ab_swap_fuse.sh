#!/bin/bash
# A/B: swap-AB K4 as one fused GEMM1+GEMM2 launch vs two launches vs the 1-SM kernel (cfg5)
out=gpurun_out/ab_swap_fuse.jsonl
: > $out
for rep in 1 2; do
  for v in 1sm unfused fused; do
    unset MOE_GEMM_VARIANT MOE_SWAP_FUSE
    case $v in 1sm) export MOE_GEMM_VARIANT=1sm;; unfused) export MOE_SWAP_FUSE=0;; esac
    timeout 300 python bench_configs.py --configs cfg5 --steps 300 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
  done
done
unset MOE_GEMM_VARIANT MOE_SWAP_FUSE
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_fused.csv python bench_configs.py --configs cfg5 --steps 5 --warmup 2 > /dev/null 2>&1
