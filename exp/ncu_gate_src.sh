#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gate_tc -s 2 -c 1 \
  -o $o/prof_gate python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu_gate.log 2>&1
ncu -i $o/prof_gate.ncu-rep --page source --csv --print-source sass > $o/src.csv 2>/dev/null
ncu -i $o/prof_gate.ncu-rep --page raw --csv > $o/raw.csv 2>/dev/null
