#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 300 python exp/gate_trace.py > $o/gate_trace.txt 2>&1; cat $o/gate_trace.txt
timeout 600 python -m pytest tests/test_gpu_gate_tc.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
