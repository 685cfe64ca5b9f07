#!/bin/bash
# cost of the 2-SM K4 epilogue stores: rebuild with -DMOE_EPI_NOSTORE=1 (outputs wrong) vs normal
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
for ns in 1 0; do
  touch paper_2603_06350_b200/csrc/kernels/ffn_gemm.cu
  make -C paper_2603_06350_b200/csrc -j16 EXTRA_NVFLAGS=-DMOE_EPI_NOSTORE=$ns > /dev/null 2>&1 || echo "build failed" >> $o/ab.txt
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "nostore=$ns" >> $o/ab.txt
  for rep in 1 2 3; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nostore=$ns bench', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], round(d.get('energy',{}).get('joules_per_step',0),2))" >> $o/ab.txt
  done
done
cat $o/ab.txt
