#!/bin/bash
# Refresh of the round-1 numbers in profiles/README.md (one B200)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench_configs.py --configs cfg1,cfg3,cfg5 --steps 200 --out gpurun_out/configs.json > /dev/null 2>&1
timeout 300 python bench_configs.py --configs cfg1,cfg5 --steps 200 --graphs --out gpurun_out/configs_graphs.json > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_swap -c 1 -o gpurun_out/swap_cfg5 \
  python bench_configs.py --configs cfg5 --steps 3 --warmup 1 > gpurun_out/ncu_swap.log 2>&1
