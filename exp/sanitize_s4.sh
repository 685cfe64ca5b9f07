#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
for sc in ${SCEN:-gatetc gatetcpred 2smbig graph}; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python profiles/sanitize_forward_r02.py $sc > $o/${sc}_${tool}.log 2>&1
    echo "$sc $tool rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' $o/${sc}_${tool}.log) $(tail -1 $o/${sc}_${tool}.log)"
  done
done
