#!/bin/bash
# K1 launch list at cfg2 (cold, serialised) + the gate tests
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate_tc -c 8 --csv --log-file $o/launches_gate.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
grep gpu__time_duration $o/launches_gate.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
