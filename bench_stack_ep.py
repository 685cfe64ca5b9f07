#!/usr/bin/env python
"""Expert-parallel MoE stack with placement-driven replica residency: does
layer-aware planning hide the replicas' cold starts?  (SURVEY.md §8f f1 + f2,
§8e; the reference's cold_start_ms, simulator.cpp:198-199, made measurable.)

  MOE_BENCH_SHARE_DEVICE=1 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 \\
      bench_stack_ep.py --layers 8          # ranks sharing one GPU (flow check)
  torchrun --nproc-per-node 8 bench_stack_ep.py --layers 8

Every rank holds only its home experts plus `--slots` replica cache slots per
layer (MOE_RESIDENCY_PLACED).  The routing drifts every `--drift` iterations
(the reference's drift re-permutation, workload.cpp:59-75), so the planner
keeps moving straggler replicas and cold replicas must be copied from their
home GPU.  Two planning modes on identical inputs:

  predicted : MoEless — layer l's fused predictor scores layer l+1, the host
              plans layer l+1 while layer l's GEMMs run, and its replica copies
              start then (they overlap layer l);
  sync      : plan on the layer's own actual loads (distance 0) — the copies
              sit on the layer's critical path.

Per mode: per-layer device latency (CUDA events on the context stream, host
running ahead, max over ranks), p50/p99, and the weight copies per layer from
one extra synchronised pass.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=4096, help="tokens per rank and layer")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--slots", type=int, default=0, help="replica cache slots per layer (0: from the memory cap)")
    ap.add_argument("--extra", type=int, default=4, help="memory cap in extra replicas per layer")
    ap.add_argument("--cap", type=int, default=0,
                    help="replicas one GPU may host per layer (gpu_mem_capacity_mb = cap x expert size; the "
                         "default cache slots follow it, so every placement the planner makes is resident)")
    ap.add_argument("--drift", type=int, default=1, help="popularity re-permutation period (iterations)")
    ap.add_argument("--modes", default="predicted,sync")
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_06350_b200 import (MOE_EXCHANGE_P2P, MOE_PLAN_PREDICTED, MOE_PLAN_SYNC, MoELayer, percentile)
    from paper_2603_06350_b200 import _capi
    from paper_2603_06350_b200 import workload as wl

    G = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("MOE_BENCH_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    if G < 2:
        print(json.dumps({"error": "run under torchrun with >= 2 ranks"}))
        return 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo" if shared else "nccl", **({} if shared else
                                                              {"device_id": torch.device("cuda", local)}))
    E, k, d, ff, s = 8, 2, 4096, 14336, 1.2
    L, T = a.layers, a.tokens
    mem = 3.0 * d * ff * 2 / 1e6
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    n_it = a.warmup + a.iters + 1
    gates = [[wl.gate_weights(E, d, s, 1, l, it, num_layers=L, drift_period=a.drift) for l in range(L)]
             for it in range(n_it)]
    xs = [torch.from_numpy(wl.tokens(T, d, E, 1, 1000 * rank + l).view(np.int16)).cuda() for l in range(L)]
    ys = [torch.empty((T, d), dtype=torch.int16, device="cuda") for _ in range(L)]
    results = {}
    for mode_name in a.modes.split(","):
        mode = MOE_PLAN_PREDICTED if mode_name == "predicted" else MOE_PLAN_SYNC
        m = MoELayer(L, E, k, d, ff, max_tokens=T, world_size=G, rank=rank, device=local,
                     exchange_mode=MOE_EXCHANGE_P2P, num_predictor_targets=1, predictor_distance=1,
                     expert_mem_mb=mem, layer_mem_cap_mb=(E + a.extra) * mem, keep_alive_iters=50,
                     gpu_mem_capacity_mb=(a.cap * mem + 1e-6) if a.cap else 180000.0,
                     residency=_capi.MOE_RESIDENCY_PLACED, replica_slots=a.slots)
        handles = [None] * G
        dist.all_gather_object(handles, m.p2p_export())
        m.p2p_import(handles)
        for l in range(L):
            for e in range(E):
                m.load_expert(l, e, *experts[e])
        stream = torch.cuda.ExternalStream(m.stream_ptr)

        def set_iteration(it):
            for l in range(L):
                m.set_gate(l, gates[it][l])
                if l + 1 < L:
                    m.set_predictor(l, 0, gates[it][l + 1])  # scores layer l+1 from layer l's input

        def barrier():
            torch.cuda.synchronize()
            dist.barrier()

        lat = []
        for it in range(a.warmup + a.iters):
            set_iteration(it)
            barrier()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
            for l in range(L):
                ev[l][0].record(stream)
                m.forward(l, xs[l], ys[l], mode, it)
                ev[l][1].record(stream)
            torch.cuda.synchronize()
            if it >= a.warmup:
                lat += [b.elapsed_time(e) for b, e in ev]
        # one synchronised pass for the copy counts (stats mode waits per layer)
        it = a.warmup + a.iters
        set_iteration(it)
        barrier()
        sts = [m.forward(l, xs[l], ys[l], mode, it, stats=True) for l in range(L)]
        barrier()
        mine = torch.tensor([statistics.mean(lat), percentile(lat, 0.5), percentile(lat, 0.99),
                             float(sum(st.weight_copies for st in sts)), float(sum(st.weight_hits for st in sts)),
                             float(sum(st.weight_copy_ms for st in sts))], dtype=torch.float64,
                            device="cpu" if shared else "cuda")
        allv = [torch.zeros_like(mine) for _ in range(G)]
        dist.all_gather(allv, mine)
        allv = torch.stack(allv).cpu().numpy()
        results[mode_name] = {
            "layer_ms_mean_max_over_ranks": float(allv[:, 0].max()), "layer_ms_p50": float(allv[:, 1].max()),
            "layer_ms_p99": float(allv[:, 2].max()),
            "weight_copies_per_iteration": [int(v) for v in allv[:, 3]],
            "warm_hits_per_iteration": [int(v) for v in allv[:, 4]],
            "copy_ms_per_iteration": [round(float(v), 3) for v in allv[:, 5]],
            "plan_sources": [st.plan_source for st in sts],
        }
        m.close()
        barrier()
    if rank == 0:
        print(json.dumps({"bench": "expert-parallel stack, placement-driven residency", "gpus": G,
                          "shared_device": shared, "layers": L, "tokens_per_rank": T,
                          "shape": {"E": E, "k": k, "d": d, "ff": ff, "zipf_s": s}, "drift_period": a.drift,
                          "replica_slots": a.slots or "from the cap", "cap_replicas_per_gpu": a.cap or None,
                          "iterations": a.iters, "modes": results}),
              flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
