#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_fused_y.py -q -x -k swap 2>&1 | tail -1
bash exp/ab_swap_combine.sh $1
