#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/dram.txt
timeout 300 python -m pytest tests/test_gpu_p2p.py -q -x -k prefill > $o/t.log 2>&1; tail -2 $o/t.log
nvidia-smi -q | grep -iE "product name|vbios|ecc mode|current.*ecc|persistence|mig mode|power limit|clocks_event" -A1 | head -40 > $o/smi.txt
for rep in 1 2 3; do
  for v in 2sm 1sm; do
    MOE_GEMM_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:grouped_gemm -s 2 -c 2 --csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "$v rep=$rep" >> $o/dram.txt
  done
done
cat $o/dram.txt
