#!/bin/bash
# 2-SM K4: DRAM bytes per launch (ncu) and tokens/s (3 x 20-step bench) per L2 policy
o=gpurun_out/$1; mkdir -p $o; : > $o/sweep.txt
shift
for p in "$@"; do
  export MOE_GEMM_L2POL=$p
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:grouped_gemm_2sm -s 2 -c 2 --csv python bench.py --steps 2 --warmup 1 --no-e2e \
    --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "pol=$p" >> $o/sweep.txt
done
for rep in 1 2 3; do
  for p in "$@"; do
    export MOE_GEMM_L2POL=$p
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pol=$p', 'bench', round(d['value']), round(d['roofline']['achieved']))" >> $o/sweep.txt
  done
done
cat $o/sweep.txt
