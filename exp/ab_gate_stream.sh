#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_predictor.py tests/test_gpu_stack.py tests/test_gpu_ids_bridge.py -q -x > $o/t.log 2>&1; tail -3 $o/t.log
for st in 0 1; do
  for rep in 1 2; do
    MOE_GATE_STREAM=$st timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_ -s 3 -c 3 --csv \
      python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg2 stream=$st" >> $o/ab.txt
    MOE_GATE_STREAM=$st timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_ -s 3 -c 3 --csv \
      python bench.py --workload cfg3 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg3 stream=$st" >> $o/ab.txt
  done
done
timeout 600 python bench_configs.py --configs cfg4 --steps 30 > $o/cfg4.json 2> $o/cfg4.err
cat $o/ab.txt; cat $o/cfg4.json | head -c 1500
