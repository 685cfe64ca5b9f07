#!/bin/bash
# A/B of programmatic dependent launch for the small per-layer kernels
# (MOE_PDL_FRONT bit mask: 1 prefix+dispatch eager, 2 combine eager, 4 / 8 the same in graphs)
out=gpurun_out/ab_pdl_front.jsonl
: > $out
for rep in 1 2; do
  for m in 0 1 3 15 5; do
    export MOE_PDL_FRONT=$m
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"variant\": \"$m\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$m\", \"rep\": $rep, /" >> $out
  done
done
