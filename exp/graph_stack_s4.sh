#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_graph_stack.py -q -x > $o/t.log 2>&1; tail -15 $o/t.log
for L in 1 4 8; do timeout 600 python bench_configs.py --configs cfg5,cfg1 --steps 200 --stack-graph $L --out $o/stack_L$L.json > /dev/null 2>&1; done
timeout 600 python bench_configs.py --configs cfg5,cfg1 --steps 300 --graphs --out $o/single.json > /dev/null 2>&1
python - <<PY
import json
for f in ["stack_L1", "stack_L4", "stack_L8", "single"]:
    try:
        for r in json.load(open("$o/%s.json" % f)):
            print(f, r["config"], round(r.get("p50_layer_ms", r.get("p50_ms", 0))*1e3, 1), round(r.get("p99_layer_ms", r.get("p99_ms", 0))*1e3, 1))
    except Exception as e: print(f, "failed", e)
PY
