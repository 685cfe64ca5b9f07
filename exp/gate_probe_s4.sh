#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 120 ./exp/gate_stream_probe > $o/probe.txt 2>&1; cat $o/probe.txt
timeout 300 python exp/gate_trace.py > $o/gate_trace.txt 2>&1; cat $o/gate_trace.txt
