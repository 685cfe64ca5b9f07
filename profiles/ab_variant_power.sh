# 1-SM vs 2-SM K4 under the board power cap (cfg2), interleaved, + DRAM/L2 bytes per launch
for v in 2sm 1sm; do
  MOE_GEMM_VARIANT=$v timeout 200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum -k regex:grouped_gemm --clock-control none -s 6 -c 4 --csv --log-file gpurun_out/var_ncu_$v.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for rep in 1 2 3; do for v in 1sm 2sm; do
  MOE_GEMM_VARIANT=$v timeout 200 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | sed "s/^/$v /"
done; done
