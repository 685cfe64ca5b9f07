#!/bin/bash
o=gpurun_out/$1; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_stack.py tests/test_gpu_residency.py tests/test_gpu_predictor.py tests/test_gpu_copy_exchange.py -q -x > $o/t.log 2>&1; tail -2 $o/t.log
for plan in sync predicted; do
  MOE_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 2 --steps 20 --warmup 5 --plan $plan --no-cpu-baseline > $o/n2_$plan.json 2> $o/n2_$plan.err
  python -c "
import json; d=json.load(open('$o/n2_$plan.json')); print('$plan', round(d['value']), d['ms_per_step'], d['p50_ms'], d['p99_ms'], d['phase_ms_median']['plan_ms'], d.get('e2e',{}).get('value'), d['config']['planner'])"
done
