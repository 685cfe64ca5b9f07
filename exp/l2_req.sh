#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/l2.txt
for v in 2sm 1sm; do
  MOE_GEMM_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:grouped_gemm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "$v" >> $o/l2.txt
done
cat $o/l2.txt
