#!/bin/bash
# Refresh of the round-1 numbers in profiles/README.md (one B200)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench_configs.py --configs cfg1,cfg3,cfg5 --steps 200 --out gpurun_out/configs.json > /dev/null 2>&1
timeout 300 python bench_configs.py --configs cfg1,cfg5 --steps 200 --graphs --out gpurun_out/configs_graphs.json > /dev/null 2>&1
timeout 600 python bench_configs.py --configs cfg4 --steps 20 --out gpurun_out/cfg4.json > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv \
  python bench_configs.py --configs cfg5 --steps 5 --warmup 2 > /dev/null 2>&1
