#!/bin/bash
# N>1 bench flow with ranks sharing one GPU (gloo plumbing, peer-memory exchange between contexts on device 0)
o=gpurun_out/$1; mkdir -p $o
for n in 2 4; do
  MOE_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n \
    bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > $o/n$n.json 2> $o/n$n.err
  python -c "
import json; d=json.loads(open('$o/n$n.json').read().strip().splitlines()[-1]); print($n, round(d['value']), d['ms_per_step'], d['p99_ms'], d.get('exchange'), d['config']['planner'], d.get('straggler_balance', d.get('balance')))"
done
MOE_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 \
    bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > $o/ref_n2.json 2> $o/ref_n2.err; tail -c 300 $o/ref_n2.json
