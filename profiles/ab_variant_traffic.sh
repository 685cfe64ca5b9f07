# DRAM / L2 bytes per K4 launch for the 1-SM and 2-SM kernels (cfg2), and the
# cfg5 decode GEMMs with and without the MMAs (data movement only: MOE_EXP=1)
for v in 1sm 2sm; do
  MOE_GEMM_VARIANT=$v timeout 200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum -k regex:grouped_gemm --clock-control none -s 6 -c 4 --csv --log-file gpurun_out/var_ncu_$v.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for v in 0 1 0 1; do MOE_EXP=$v timeout 200 python bench_configs.py --configs cfg5 --steps 30 --warmup 5 2>/dev/null | sed "s/^/exp$v /"; done
