#!/usr/bin/env python
"""Per-config measurements beside the headline bench (one B200).

  python bench_configs.py [--configs cfg1,cfg3,cfg5] [--steps 50] [--warmup 5]

For each BASELINE.json config that fits one GPU: layer latency p50/p99
(nearest rank, device events, host running ahead), tokens/s, the phase
breakdown and the K4 roofline; rows are re-routed every step.  The multi-GPU
configs (cfg3 at G=2/4/8, cfg4, cfg5 at G=8) are run here at G=1 with the same
per-GPU shapes and labelled so; bench.py --gpus N covers the EP path.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def run_config(name, steps, warmup, graphs=False):
    import numpy as np
    import torch

    from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer, percentile
    from paper_2603_06350_b200 import workload as wl
    c = dict(wl.CONFIGS[name])
    E, k, d, ff, T, s = c["E"], c["k"], c["d"], c["ff"], c["T"], c["s"]
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=c["extra_replicas"] * mem,
                 cuda_graphs=graphs)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
    n_it = warmup + steps + 10
    gates = torch.from_numpy(np.stack([wl.gate_weights(E, d, s, 1, 0, it)
                                       for it in range(n_it)]).view(np.int16)).cuda()
    y = torch.empty((T, d), dtype=torch.int16, device="cuda")
    stream = torch.cuda.ExternalStream(m.stream_ptr)

    # the layer reads a static input buffer, refilled from the pool before each
    # step (as a serving engine feeds its captured decode graph): one CUDA graph
    # per (layer, tokens, buffers) is replayed; cycling graph executables per
    # pool buffer instead costs ~6 us per launch (profiles/ab_graph_stack_r02.md)
    x_static = torch.empty_like(pool[0])

    def step(it, stats=False, ev_start=None):
        # device-resident per-iteration gates re-route every step; the gate and
        # token uploads are not part of the layer (K1 .. K5), so the layer's start
        # event follows them
        with torch.cuda.stream(stream):
            x_static.copy_(pool[it % 4])
        m.set_gate_device(0, gates[it])
        if ev_start is not None:
            ev_start.record(stream)
        return m.forward(0, x_static, y, MOE_PLAN_SYNC, it, stats=stats)

    for it in range(warmup):
        step(it)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(steps):
        step(warmup + i, ev_start=ev[i][0])
        ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) for a, b in ev]
    total = t0.elapsed_time(t1)
    st = [step(warmup + steps + i, stats=True) for i in range(10)]
    phases = {p: statistics.median(getattr(x, p) for x in st)
              for p in ("gate_ms", "plan_ms", "dispatch_ms", "gemm1_ms", "gemm2_ms", "combine_ms")}
    rows = statistics.median(x.rows_local for x in st)
    flops = 6.0 * d * ff * rows
    gemm = phases["gemm1_ms"] + phases["gemm2_ms"]
    active = statistics.median(sum(1 for e in range(E) if x.counts[e] > 0) for x in st)
    wbytes = active * 3 * d * ff * 2
    m.close()
    return {
        "config": name, "shape": c, "tokens_per_s": T * steps / (total * 1e-3), "ms_per_step": total / steps,
        "p50_ms": percentile(lat, 0.5), "p99_ms": percentile(lat, 0.99), "phase_ms_median": phases,
        "k4_tflops": flops / (gemm * 1e-3) / 1e12, "k4_weight_gbs": wbytes / (gemm * 1e-3) / 1e9,
        "active_experts": active, "replicas_median": statistics.median(x.replica_count for x in st),
        "gpus": 1, "note": "per-GPU shape at G=1" if c["G"] > 1 else "", "cuda_graphs": graphs,
    }


def run_graph_stack(name, n_layers, steps, warmup):
    """A decode step over `n_layers` layers of the named shape recorded as ONE CUDA
    graph (moe_graph_begin / moe_graph_end; one graph launch per step, as a serving
    engine replays a whole decode step): per-layer latency = graph time / n_layers.
    Every layer has its own expert weights in HBM (1.07 GB each at cfg5, far above
    L2) and its own gate, re-routed every step by device-to-device gate updates
    that sit outside the timed window; layer inputs are independent synthetic
    batches (the routing statistics of the single-layer config)."""
    import numpy as np
    import torch

    from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer, percentile
    from paper_2603_06350_b200 import workload as wl
    c = dict(wl.CONFIGS[name])
    E, k, d, ff, T, s = c["E"], c["k"], c["d"], c["ff"], c["T"], c["s"]
    m = MoELayer(n_layers, E, k, d, ff, max_tokens=T)
    host_experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    for l in range(n_layers):  # same values, separate HBM copies per layer
        for e in range(E):
            m.load_expert(l, e, *host_experts[e])
    pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
    ys = [torch.empty((T, d), dtype=torch.int16, device="cuda") for _ in range(n_layers)]
    n_gate_sets = 16
    gates = torch.from_numpy(np.stack([np.stack([wl.gate_weights(E, d, s, 1, l, g) for l in range(n_layers)])
                                       for g in range(n_gate_sets)]).view(np.int16)).cuda()
    stream = torch.cuda.ExternalStream(m.stream_ptr)

    def set_gates(it):
        for l in range(n_layers):
            m.set_gate_device(l, gates[it % n_gate_sets, l])

    set_gates(0)
    m.graph_begin()
    for l in range(n_layers):
        m.forward(l, pool[l % 4], ys[l], MOE_PLAN_FIXED, 0)
    gid = m.graph_end()
    for it in range(warmup):
        set_gates(it)
        m.graph_launch(gid)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        set_gates(warmup + i)
        ev[i][0].record(stream)
        m.graph_launch(gid)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    per_layer = [t / n_layers for t in step_ms]
    m.close()
    return {
        "config": name, "mode": "graph_stack", "layers": n_layers, "shape": c, "steps": steps,
        "p50_layer_ms": percentile(per_layer, 0.5), "p99_layer_ms": percentile(per_layer, 0.99),
        "p50_step_ms": percentile(step_ms, 0.5), "p99_step_ms": percentile(step_ms, 0.99),
        "tokens_per_s_per_layer": T * n_layers * steps / (sum(step_ms) * 1e-3), "gpus": 1,
        "note": "per-GPU shape at G=1; one CUDA graph of %d layer forwards per step (moe_graph_begin/end), "
                "per-layer = graph time / layers; gate re-routing uploads outside the window" % n_layers,
    }


def run_stack(name, iters, warmup, layers=None):
    """cfg4: the 32-layer Mixtral-shape MoE stack with the layer-aware predictor
    and planner-driven scaling/placement (MOE_PLAN_PREDICTED, distance 1)."""
    import numpy as np
    import torch

    from paper_2603_06350_b200 import percentile
    from paper_2603_06350_b200 import workload as wl
    from paper_2603_06350_b200.stack import MoEStack
    c = dict(wl.CONFIGS[name])
    L = layers or c.get("L", 32)
    E, k, d, ff, T = c["E"], c["k"], c["d"], c["ff"], c["T"]
    st = MoEStack(L, E, k, d, ff, T, extra_replicas=c["extra_replicas"], zipf_s=c["s"], distance=1)
    pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
    y = torch.empty((T, d), dtype=torch.int16, device="cuda")
    hs = [torch.empty((T, d), dtype=torch.int16, device="cuda") for _ in range(2)]  # residual stream
    stream = torch.cuda.ExternalStream(st.layer.stream_ptr)

    def run_iteration(it, stats=False, ev_row=None):
        # The residual stream of a real stack: layer l + 1 reads h + y of layer l (bf16 add on
        # the layer's stream), so layer l's fused predictor scores layer l + 1 on the hidden
        # state the next layer actually sees, one residual update earlier.
        x, out = pool[it % 4], []
        with torch.cuda.stream(stream):
            for l in range(L):
                if ev_row is not None:
                    ev_row[l][0].record(stream)
                r = st.layer.forward(l, x, y, 2, it, stats=stats)
                if ev_row is not None:
                    ev_row[l][1].record(stream)
                out.append(r)
                h = hs[l % 2]
                torch.add(x.view(torch.bfloat16), y.view(torch.bfloat16), out=h.view(torch.bfloat16))
                x = h
        return out

    for it in range(warmup):
        run_iteration(it)
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
          for _ in range(iters)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(iters):
        run_iteration(warmup + i, ev_row=ev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) for row in ev for a, b in row]  # all (iteration, layer) samples (MoE layer only)
    total = t0.elapsed_time(t1)
    stats = run_iteration(warmup + iters, stats=True)
    acc = [s.predictor_accuracy for s in stats[1:]]
    res = {
        "config": name, "layers": L, "gpus": 1, "shape": c, "iterations": iters,
        "ms_per_stack": total / iters, "ms_per_layer_mean": total / iters / L,
        "p50_layer_ms": percentile(lat, 0.5), "p99_layer_ms": percentile(lat, 0.99),
        "tokens_per_s_per_layer": T * iters * L / (total * 1e-3),
        "predictor_accuracy_mean": sum(acc) / len(acc), "predictor_accuracy_min": min(acc),
        "plan_sources": [s.plan_source for s in stats], "replicas": [s.replica_count for s in stats],
        "note": "per-GPU shape at G=1 (named config is G=8); planning from the fused predictor, distance 1; "
                "layers chained through the residual stream h_{l+1} = h_l + y_l (ms_per_stack includes the adds, "
                "the layer samples do not)",
    }
    st.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg3,cfg5")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default="")
    ap.add_argument("--graphs", action="store_true", help="replay single-GPU forwards as CUDA graphs")
    ap.add_argument("--stack-graph", type=int, default=0,
                    help="record this many layers of each config as one CUDA graph per step (decode stack)")
    a = ap.parse_args()
    if a.stack_graph:
        res = [run_graph_stack(n, a.stack_graph, a.steps, a.warmup) for n in a.configs.split(",")]
    else:
        res = [run_stack(n, max(2, a.steps // 10), 1) if n == "cfg4" else run_config(n, a.steps, a.warmup, a.graphs)
               for n in a.configs.split(",")]
    for r in res:
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
