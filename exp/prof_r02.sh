#!/bin/bash
# round-2 evidence: GPU tests, bench (both arms), launch list and a full capture of the K4 kernels
o=gpurun_out/r02k; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q > $o/gputests.log 2>&1; tail -3 $o/gputests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > $o/bench200.json 2> $o/bench200.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_2sm -s 2 -c 2 \
  -o $o/prof_gemm python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"gate_topk|dispatch_kernel|combine_kernel" -s 3 -c 3 \
  -o $o/prof_small python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_small.log 2>&1
ls -la $o
