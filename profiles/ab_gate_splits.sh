#!/bin/bash
# K1 split-K bound at the decode shape (cfg5: 8 blocks of 32 tokens)
out=gpurun_out/ab_gate_splits.jsonl
: > $out
for rep in 1 2; do
  for sp in 16 8 4 2; do
    export MOE_GATE_MAX_SPLITS=$sp
    timeout 300 python bench_configs.py --configs cfg5 --steps 300 | sed "s/^{/{\"variant\": \"$sp\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$sp\", \"rep\": $rep, /" >> $out
  done
done
