#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gate_|block_prefix|dispatch_kernel|combine_kernel" -s 10 -c 5 \
  -o $o/prof_front python bench.py --workload cfg5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $o/ncu_front.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg5.csv \
  python bench_configs.py --configs cfg5 --steps 5 --warmup 2 --graphs > /dev/null 2>&1
ls -la $o
