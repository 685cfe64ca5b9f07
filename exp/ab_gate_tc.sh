#!/bin/bash
# prefill gate: tcgen05 + TMA (MOE_GATE_TC=1) vs per-block mma.sync (0), same box
o=gpurun_out/$1; mkdir -p $o; : > $o/bench.jsonl
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py tests/test_gpu_stack.py -q -x > $o/t.log 2>&1; tail -3 $o/t.log
for rep in 1 2; do
  for tc in 0 1; do
    MOE_GATE_TC=$tc timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | sed "s/^{/{\"tc\": $tc, \"rep\": $rep, /" >> $o/bench.jsonl
  done
done
python -c "
import json
for l in open('$o/bench.jsonl'):
    d=json.loads(l); print(d['tc'], d['rep'], round(d['value']), 'gate_ms', round(d['phase_ms_median']['gate_ms']*1e3,1), 'step', round(d['ms_per_step'],3))"
for tc in 0 1; do
MOE_GATE_TC=$tc timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gate -c 6 --csv --log-file $o/gate_$tc.csv python bench.py --steps 3 --warmup 1 > /dev/null 2>&1
python exp/ncu_csv.py gate$tc < $o/gate_$tc.csv
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gate_tc -s 2 -c 1 -o $o/gate_tc_full python bench.py --steps 3 --warmup 1 > /dev/null 2>&1
ls $o
