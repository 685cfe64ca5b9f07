#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_gate_tc.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for b in 1 2 4; do MOE_GATE_TC_BKS=$b timeout 300 python -m pytest tests/test_gpu_gate_tc.py -q -x 2>&1 | tail -1; done
for b in 1 2 4; do
MOE_GATE_TC_BKS=$b timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg --clock-control none -k regex:gate -c 6 --csv --log-file $o/gate_b$b.csv python bench.py --steps 3 --warmup 1 > /dev/null 2>&1
python exp/ncu_csv.py bks$b < $o/gate_b$b.csv
done
MOE_GATE_TC=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg --clock-control none -k regex:gate -c 4 --csv --log-file $o/gate_old.csv python bench.py --steps 3 --warmup 1 > /dev/null 2>&1
python exp/ncu_csv.py old < $o/gate_old.csv
