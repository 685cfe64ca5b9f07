#!/bin/bash
# A/B: L2 policy of the swap-AB weight stream (0 evict_last, 1 evict_first, 2 evict_normal)
out=gpurun_out/ab_swap_wpol.jsonl
: > $out
for rep in 1 2; do
  for w in 0 1 2; do
    export MOE_SWAP_WPOL=$w
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"variant\": \"$w\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$w\", \"rep\": $rep, /" >> $out
  done
done
