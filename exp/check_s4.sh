#!/bin/bash
# session-4 baseline check: GPU suite, smoke, headline bench, decode graphs
o=gpurun_out/$1; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > $o/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $o/gputests.log 2>&1; tail -2 $o/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
timeout 600 python bench_configs.py --configs cfg1,cfg5 --steps 300 --graphs --out $o/configs_graphs.json > /dev/null 2>&1
ls $o
