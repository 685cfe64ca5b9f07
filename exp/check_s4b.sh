#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x > $o/gputests.log 2>&1; tail -2 $o/gputests.log
timeout 600 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs --out $o/configs_graphs.json > /dev/null 2>&1
timeout 600 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 200 --stack-graph 8 --out $o/stack8.json > /dev/null 2>&1
python - <<PY
import json
for f in ["configs_graphs", "stack8"]:
    for r in json.load(open("$o/%s.json" % f)):
        print(f, r["config"], round(r.get("p50_layer_ms", r.get("p50_ms", 0))*1e3, 1), round(r.get("p99_layer_ms", r.get("p99_ms", 0))*1e3, 1))
PY
