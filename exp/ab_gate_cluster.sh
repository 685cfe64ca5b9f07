#!/bin/bash
# A/B of the split-K gate reduction: cluster (DSMEM, one launch) vs finish kernel,
# at the decode shapes (graph-replayed and eager) and cfg2 with split 2 forced.
o=gpurun_out/$1; mkdir -p $o; out=$o/ab.jsonl; : > $out
timeout 300 python -m pytest tests/test_gpu_layer.py tests/test_gpu_predictor.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for rep in 1 2; do
  for cl in 0 1; do
    export MOE_GATE_CLUSTER=$cl
    timeout 300 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs | sed "s/^{/{\"cluster\": $cl, \"rep\": $rep, \"graphs\": 1, /" >> $out
    timeout 300 python bench_configs.py --configs cfg5,cfg1 --steps 300 | sed "s/^{/{\"cluster\": $cl, \"rep\": $rep, \"graphs\": 0, /" >> $out
  done
  for ms in 1 2 4; do
    MOE_GATE_MIN_SPLITS=$ms timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(min_splits=$ms, rep=$rep, tok_s=d['value'], gate_ms=d['phase_ms_median']['gate_ms'])))" >> $out
  done
done
cat $out | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:d.get(k) for k in ('cluster','rep','graphs','config','p50_ms','p99_ms','min_splits','tok_s','gate_ms') if k in d})"
