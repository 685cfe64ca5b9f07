#!/bin/bash
# A/B of two builds of libmoe_b200.so on the same box (exp/_old_lib = previous commit; not tracked)
out=gpurun_out/ab_old_new.jsonl
: > $out
cp paper_2603_06350_b200/libmoe_b200.so /tmp/lib_new.so
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp exp/_old_lib/libmoe_b200.so paper_2603_06350_b200/libmoe_b200.so; else cp /tmp/lib_new.so paper_2603_06350_b200/libmoe_b200.so; fi
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $out
  done
done
cp /tmp/lib_new.so paper_2603_06350_b200/libmoe_b200.so
