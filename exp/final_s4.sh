#!/bin/bash
# session-4 evidence refresh with the current defaults
o=gpurun_out/$1; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > $o/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $o/gputests.log 2>&1; tail -2 $o/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $o/ref.json 2> $o/ref.err
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > $o/bench200.json 2> $o/bench200.err
timeout 900 python bench_configs.py --configs cfg1,cfg3,cfg5,cfg5s12 --steps 200 --out $o/configs.json > /dev/null 2>&1
timeout 600 python bench_configs.py --configs cfg1,cfg5,cfg5s12 --steps 300 --graphs --out $o/configs_graphs.json > /dev/null 2>&1
timeout 900 python bench_configs.py --configs cfg4 --steps 30 --out $o/cfg4.json > /dev/null 2>&1
timeout 600 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 200 --stack-graph 8 --out $o/stack8.json > /dev/null 2>&1
timeout 300 python exp/gate_trace.py > $o/gate_trace.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $o/launches_cfg5.csv \
  python bench_configs.py --configs cfg5 --steps 10 --warmup 2 --graphs > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_2sm -s 2 -c 2 \
  -o $o/prof_gemm python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gate_tc|dispatch_kernel|combine_kernel" -s 3 -c 3 \
  -o $o/prof_small python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_small.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"frontend_kernel|grouped_gemm_swap" -s 4 -c 2 \
  -o $o/prof_decode python bench_configs.py --configs cfg5 --steps 3 --warmup 2 > $o/ncu_decode.log 2>&1
ls $o
