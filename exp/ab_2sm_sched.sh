#!/bin/bash
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
timeout 300 python -m pytest tests/test_gpu_gemm_variants.py tests/test_gpu_p2p.py -q -x -k "agree or prefill" > $o/t.log 2>&1; tail -2 $o/t.log
for sch in static dynamic; do
  MOE_GEMM_SCHED=$sch timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum --clock-control none -k regex:grouped_gemm -s 2 -c 2 --csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python exp/ncu_csv.py "$sch" >> $o/ab.txt
done
for rep in 1 2 3; do
  for sch in static dynamic; do
    MOE_GEMM_SCHED=$sch timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sch', 'bench', round(d['value']), round(d['roofline']['achieved']))" >> $o/ab.txt
  done
done
cat $o/ab.txt
