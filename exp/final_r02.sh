#!/bin/bash
# round-2 evidence refresh with the final defaults
o=gpurun_out/$1; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q > $o/gputests.log 2>&1; tail -2 $o/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $o/ref.json 2> $o/ref.err
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > $o/bench200.json 2> $o/bench200.err
timeout 900 python bench_configs.py --configs cfg1,cfg3,cfg5,cfg5s12 --steps 200 --out $o/configs.json > /dev/null 2>&1
timeout 600 python bench_configs.py --configs cfg1,cfg5,cfg5s12 --steps 200 --graphs --out $o/configs_graphs.json > /dev/null 2>&1
timeout 900 python bench_configs.py --configs cfg4 --steps 30 --out $o/cfg4.json > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg2" > $o/gemm_dram.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_2sm -s 2 -c 2 \
  -o $o/prof_gemm python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"gate_topk|dispatch_kernel|combine_kernel" -s 3 -c 3 \
  -o $o/prof_small python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_small.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"grouped_gemm_swap" -s 3 -c 1 \
  -o $o/prof_swap python bench_configs.py --configs cfg5 --steps 3 --warmup 2 > $o/ncu_swap.log 2>&1
ls $o
