#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 300 ncu --set full --warp-sampling-interval 0 --import-source on -k regex:"gate_finish|dispatch_kernel|combine_kernel|gate_topk" -s 8 -c 4 \
  -o $o/prof_dec python bench_configs.py --configs cfg5 --steps 3 --warmup 2 > $o/ncu.log 2>&1
ls -la $o
