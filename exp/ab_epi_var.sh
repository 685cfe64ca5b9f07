#!/bin/bash
# 2-SM K4 epilogue variants under ncu: time, SM clock, tensor-pipe activity, DRAM bytes
# (the diagnostic flags of session 4 — MOE_EPI_SCRATCH, MOE_DIAG_A_SAME / B_SAME, MOE_DIAG_RED, MOE_EPI_STREAM,
#  MOE_EPI_PACE_NS — were removed from ffn_gemm.cu after the runs; results in profiles/ab_epi_store_r02.md)
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
for fl in "-DMOE_EPI_STAGED=1" "-DMOE_EPI_SCRATCH=4" "-DMOE_EPI_STAGED=1" "-DMOE_EPI_SCRATCH=4"; do
  touch paper_2603_06350_b200/csrc/kernels/ffn_gemm.cu
  make -C paper_2603_06350_b200/csrc -j16 EXTRA_NVFLAGS="$fl" > /dev/null 2>&1 || echo "build failed" >> $o/ab.txt
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "$fl" >> $o/ab.txt
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$fl bench', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])" >> $o/ab.txt
done
cat $o/ab.txt
touch paper_2603_06350_b200/csrc/kernels/ffn_gemm.cu; make -C paper_2603_06350_b200/csrc -j16 > /dev/null 2>&1
