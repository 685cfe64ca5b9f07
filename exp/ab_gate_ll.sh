#!/bin/bash
# same-box A/B of K1 at cfg2: ncu launch list (gpu__time_duration only), working tree vs exp/_old swapped in
o=gpurun_out/$1; mkdir -p $o
rm -rf /tmp/old && mkdir -p /tmp/old && cp -r . /tmp/old/ 2>/dev/null
(cd exp/_old && find . -type f -exec cp {} /tmp/old/{} \;)
(cd /tmp/old && make -C paper_2603_06350_b200/csrc -j16 > /tmp/old/build.log 2>&1) || echo "old build failed"
for rep in 1 2 3; do
  for v in old new; do
    dir=.; [ $v = old ] && dir=/tmp/old
    (cd $dir && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate_tc -c 6 --csv --log-file /tmp/ll_$v.csv \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1)
    echo "$v $rep: $(grep gpu__time_duration /tmp/ll_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')" | tee -a $o/ab.txt
  done
done
