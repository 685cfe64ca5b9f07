#!/bin/bash
# 2-SM GEMM2 writing y directly (MOE_FUSED_Y=1, default) vs yp + combine kernel (MOE_FUSED_Y=0)
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
for fy in 1 0; do
  MOE_FUSED_Y=$fy timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"grouped_gemm_2sm|combine" -s 3 -c 3 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "fy=$fy" >> $o/ab.txt
done
for rep in 1 2 3; do
for fy in 1 0; do
  MOE_FUSED_Y=$fy timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fy=$fy bench', round(d['value']), round(d['e2e']['value']), round(d['p99_ms'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['gpu_launches'])" >> $o/ab.txt
done
done
cat $o/ab.txt
