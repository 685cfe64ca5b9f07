#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
timeout 300 python exp/gate_trace.py 2>&1 | tail -3
bash exp/ab_gate_ll.sh $1
