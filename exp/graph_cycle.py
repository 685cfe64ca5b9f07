"""cfg5 single-layer CUDA-graph replays through moe_graph_begin/end: one graph
replayed vs four graphs (one per input buffer) cycled, as the per-forward
graph cache does for bench_configs' 4-buffer token pool."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer, percentile
from paper_2603_06350_b200 import workload as wl

c = dict(wl.CONFIGS["cfg5"])
E, k, d, ff, T, s = c["E"], c["k"], c["d"], c["ff"], c["T"], c["s"]
m = MoELayer(1, E, k, d, ff, max_tokens=T)
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
gates = torch.from_numpy(np.stack([wl.gate_weights(E, d, s, 1, 0, it) for it in range(16)]).view(np.int16)).cuda()
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
stream = torch.cuda.ExternalStream(m.stream_ptr)
gids = []
m.set_gate_device(0, gates[0])
for i in range(4):
    m.graph_begin(); m.forward(0, pool[i], y, MOE_PLAN_FIXED, 0); gids.append(m.graph_end())
for name, pick in (("one graph", lambda i: gids[0]), ("four graphs cycled", lambda i: gids[i % 4]), ("one graph again", lambda i: gids[0])):
    for it in range(20):
        m.set_gate_device(0, gates[it % 16]); m.graph_launch(pick(it))
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
    for i in range(300):
        m.set_gate_device(0, gates[i % 16]); ev[i][0].record(stream); m.graph_launch(pick(i)); ev[i][1].record(stream)
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"{name}: p50 {percentile(lat, .5):.1f} p99 {percentile(lat, .99):.1f} us")
