#!/bin/bash
# A/B of K4 variants in the driver's regime (20 timed steps after 5 warm-ups), interleaved.
out=gpurun_out/$1; mkdir -p $out; shift
for rep in 1 2 3; do
  for v in "$@"; do
    MOE_GEMM_VARIANT=$v python bench.py --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(v='$v', rep=$rep, tok_s=d['value'], ms=d['ms_per_step'], k4=d['roofline']['achieved'], mhz=d['clocks']['sm_mhz'], j=d.get('energy',{}).get('joules_per_step'))))" >> $out/ab.jsonl
  done
done
cat $out/ab.jsonl
