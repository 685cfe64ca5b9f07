#!/bin/bash
# A/B: swap-AB GEMM1 gathering its rows from x (dispatch only ranks) vs the dispatch copy
out=gpurun_out/ab_swap_gather.jsonl
: > $out
for rep in 1 2; do
  for g in 0 1; do
    export MOE_SWAP_GATHER=$g
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"variant\": \"$g\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$g\", \"rep\": $rep, /" >> $out
  done
done
