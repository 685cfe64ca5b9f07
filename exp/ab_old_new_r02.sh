#!/bin/bash
# same-box A/B: the working tree vs the working tree with the files under exp/_old/<path> swapped in (rebuilt in /tmp/old)
o=gpurun_out/$1; mkdir -p $o; : > $o/cfg.jsonl
rm -rf /tmp/old && mkdir -p /tmp/old && cp -r . /tmp/old/ 2>/dev/null
(cd exp/_old && find . -type f -exec cp {} /tmp/old/{} \;)
(cd /tmp/old && make -C paper_2603_06350_b200/csrc -j16 > /tmp/old/build.log 2>&1) || echo "old build failed"
timeout 300 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_ids_bridge.py tests/test_gpu_p2p.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for rep in 1 2 3; do
  for v in old new; do
    dir=.; [ $v = old ] && dir=/tmp/old
    (cd $dir && timeout 300 python bench_configs.py --configs cfg5,cfg5s12,cfg1 --steps 300 --graphs) | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> $o/cfg.jsonl
  done
done
python -c "
import json
for l in open('$o/cfg.jsonl'):
    d=json.loads(l); print(d['v'], d['rep'], d['config'], round(d['p50_ms']*1e3,1), round(d['p99_ms']*1e3,1))"
