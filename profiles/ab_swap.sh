#!/bin/bash
# A/B of the swap-AB decode K4 against the 1-SM kernel on cfg5 (and cfg1 as a control)
set -x
out=gpurun_out/ab_swap.jsonl
: > $out
for rep in 1 2; do
  for v in 1sm auto; do
    if [ $v = auto ]; then unset MOE_GEMM_VARIANT; else export MOE_GEMM_VARIANT=$v; fi
    python bench_configs.py --configs cfg5,cfg1 --steps 200 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
    python bench_configs.py --configs cfg5 --steps 200 --graphs | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
  done
done
unset MOE_GEMM_VARIANT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/launches_cfg5_swap.csv python bench_configs.py --configs cfg5 --steps 5 --warmup 2 > /dev/null 2>&1
MOE_GEMM_VARIANT=1sm ncu --metrics gpu__time_duration.sum --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/launches_cfg5_1sm.csv python bench_configs.py --configs cfg5 --steps 5 --warmup 2 > /dev/null 2>&1
