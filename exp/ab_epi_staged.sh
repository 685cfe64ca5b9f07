#!/bin/bash
# 2-SM K4 epilogue: smem-staged line-coalesced stores (default) vs direct per-lane row stores
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_gemm_variants.py tests/test_gpu_ids_bridge.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for st in 0 1; do
  touch paper_2603_06350_b200/csrc/kernels/ffn_gemm.cu
  make -C paper_2603_06350_b200/csrc -j16 EXTRA_NVFLAGS=-DMOE_EPI_STAGED=$st > /dev/null 2>&1 || echo "build failed" >> $o/ab.txt
  [ $rep = 1 ] && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "staged=$st" >> $o/ab.txt
  for r2 in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('staged=$st bench', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], round(d.get('energy',{}).get('joules_per_step',0),2))" >> $o/ab.txt
  done
done
done
cat $o/ab.txt
touch paper_2603_06350_b200/csrc/kernels/ffn_gemm.cu; make -C paper_2603_06350_b200/csrc -j16 > /dev/null 2>&1
