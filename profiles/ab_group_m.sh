set -x
for rep in 1 2; do
for g in "32,16" "32,8" "32,4" "32,32" "16,16" "64,16"; do
  MOE_GEMM_GROUP_M=$g timeout 200 python bench.py --steps 60 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/gm_${g/,/_}_$rep.json 2>/dev/null
done
done
for g in "32,16" "32,8" "32,4" "32,32" "16,16" "64,16"; do
  MOE_GEMM_GROUP_M=$g timeout 200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum -k regex:grouped_gemm -s 6 -c 4 --csv --log-file gpurun_out/gm_ncu_${g/,/_}.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
