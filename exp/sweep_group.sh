#!/bin/bash
# 2-SM K4 sweep: L2 policies (MOE_GEMM_L2POL) and rasterisation (MOE_GEMM_GROUP_M=g1,g2)
o=gpurun_out/$1; mkdir -p $o; : > $o/sweep.txt
run() {  # $1 label; env already exported
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null \
    | grep grouped_gemm | awk -F'","' -v g="$1" '{gsub(/"/,"",$NF); print g, substr($5,1,30), $(NF-2), $NF}' >> $o/sweep.txt
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'bench', round(d['value']), round(d['roofline']['achieved']))" >> $o/sweep.txt
}
for p in 68 17 153 136 0 85; do export MOE_GEMM_L2POL=$p; run "pol=$p"; done
unset MOE_GEMM_L2POL
for g in "32,8" "32,4" "32,32" "16,16" "64,16"; do export MOE_GEMM_GROUP_M=$g; run "group=$g"; done
cat $o/sweep.txt
