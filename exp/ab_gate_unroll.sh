#!/bin/bash
# K1 unroll A/B: rebuild with -DMOE_GATE_UNROLL=N on the box, launch list of cfg2 + cfg5
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt; shift
for u in "$@"; do
  touch paper_2603_06350_b200/csrc/kernels/gate.cu
  make -C paper_2603_06350_b200/csrc -j8 EXTRA_NVFLAGS=-DMOE_GATE_UNROLL=$u > /dev/null 2>&1 || { echo "build $u failed" >> $o/ab.txt; continue; }
  for rep in 1 2; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_ -s 3 -c 4 --csv \
      python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg2 unroll=$u" >> $o/ab.txt
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate_ -s 6 -c 6 --csv \
      python bench.py --workload cfg5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "cfg5 unroll=$u" >> $o/ab.txt
  done
done
touch paper_2603_06350_b200/csrc/kernels/gate.cu; make -C paper_2603_06350_b200/csrc -j8 > /dev/null 2>&1
cat $o/ab.txt
