#!/bin/bash
# same-box A/B of the session-4 kernels (tree top-k K1, staged K4 epilogue) vs the session start (exp/_old)
o=gpurun_out/$1; mkdir -p $o; : > $o/ab.txt
rm -rf /tmp/old && mkdir -p /tmp/old && cp -r . /tmp/old/ 2>/dev/null
(cd exp/_old && find . -type f -exec cp {} /tmp/old/{} \;)
(cd /tmp/old && make -C paper_2603_06350_b200/csrc -j16 > /tmp/old/build.log 2>&1) || echo "old build failed"
for rep in 1 2 3; do
  for v in old new; do
    dir=.; [ $v = old ] && dir=/tmp/old
    (cd $dir && timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline) \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', $rep, round(d['value']), round(d['e2e']['value']), round(d['p99_ms'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])" >> $o/ab.txt
  done
done
cat $o/ab.txt
