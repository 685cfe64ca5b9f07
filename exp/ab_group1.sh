#!/bin/bash
# 2-SM K4 GEMM1 rasterisation: m-tiles per n sweep (MOE_GEMM_GROUP_M="g1,g2", 128-row units)
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
for rep in 1 2; do
for g in "32,16" "16,16" "64,16" "24,16"; do
  MOE_GEMM_GROUP_M=$g timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "g=$g" >> $o/ab.txt
  MOE_GEMM_GROUP_M=$g timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('g=$g bench', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])" >> $o/ab.txt
done
done
cat $o/ab.txt
