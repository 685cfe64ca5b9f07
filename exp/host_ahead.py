"""Is the host ahead of the GPU in bench_configs' single-layer graph loop (cfg5)?
Host time per m.forward call (flush of the previous forward's planner work +
graph launch) vs the device layer time, for SYNC and FIXED planning."""
import os, sys, time, statistics
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer, percentile
from paper_2603_06350_b200 import workload as wl

c = dict(wl.CONFIGS["cfg5"])
E, k, d, ff, T, s = c["E"], c["k"], c["d"], c["ff"], c["T"], c["s"]
mem = 3.0 * d * ff * 2 / 1e6
m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=c["extra_replicas"] * mem, cuda_graphs=os.environ.get("G", "1") == "1")
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
gates = torch.from_numpy(np.stack([wl.gate_weights(E, d, s, 1, 0, it) for it in range(64)]).view(np.int16)).cuda()
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
stream = torch.cuda.ExternalStream(m.stream_ptr)
for mode, name in ((MOE_PLAN_SYNC, "sync"), (MOE_PLAN_FIXED, "fixed")):
    for it in range(10):
        m.set_gate_device(0, gates[it % 64]); m.forward(0, pool[it % 4], y, mode, it)
    torch.cuda.synchronize()
    n = 300
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    fwd_us, step_us = [], []
    t_prev = time.perf_counter()
    for i in range(n):
        it = 10 + i
        m.set_gate_device(0, gates[it % 64])
        ev[i][0].record(stream)
        t0 = time.perf_counter()
        m.forward(0, pool[it % 4], y, mode, it)
        t1 = time.perf_counter()
        ev[i][1].record(stream)
        fwd_us.append((t1 - t0) * 1e6)
        step_us.append((t1 - t_prev) * 1e6)
        t_prev = t1
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"{name}: device p50 {percentile(lat, .5):.1f} us; host forward() p50 {statistics.median(fwd_us):.1f} us, "
          f"host step p50 {statistics.median(step_us):.1f} us")
