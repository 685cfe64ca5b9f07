"""Phase stamps of the tcgen05 prefill gate (MOE_FRONT_TRACE=1) at cfg2:
median over forwards of (min, max) over CTAs, us from the earliest CTA start."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MOE_FRONT_TRACE"] = "1"
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

E, k, d, T = 8, 2, 4096, 16384
m = MoELayer(1, E, k, d, 256, max_tokens=T)
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, 256, 1, 0, e))
m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
xs = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(2)]
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
names = ["prologue", "first stage", "last stage", "epilogue", "end", "epi wake", "tmem ld", "epi select", "mma commit"]
rows = []
deltas = []
cyc = []
for it in range(12):
    m.forward(0, xs[it % 2], y, MOE_PLAN_FIXED, it)
    torch.cuda.synchronize()
    tr = m.read_buffer(12, np.uint64, (148, 16)).astype(np.int64)
    n = int((tr[:, 0] > 0).sum())
    tr = tr[:n]
    t0 = tr[:, 0].min()
    cyc.append(np.median(np.stack([tr[:, 14] - tr[:, 13], tr[:, 15] - tr[:, 14]], axis=1), axis=0))
    deltas.append(np.stack([tr[:, j] - tr[:, 3] for j in (9, 6, 7, 11, 12, 8, 4, 5)], axis=1) / 1e3)
    rows.append([(tr[:, i].min() - t0, tr[:, i].max() - t0) for i in range(10)])
r = np.median(np.array(rows[2:], dtype=np.float64), axis=0) / 1e3
print(f"gate_tc cfg2: {n} CTAs; start spread {r[0][1]:.2f} us")
for i, nm in enumerate(names):
    print(f"  {nm:12s} min {r[i + 1][0]:6.2f}  max {r[i + 1][1]:6.2f} us")
# per-CTA deltas from its own last stage (median over CTAs and forwards)
print("per-CTA delta from last stage (median):", {nm: round(float(v), 2) for nm, v in zip(["mma commit", "epi wake", "tmem ld", "topk", "writes", "epi select", "epilogue", "end"], np.median(np.array(deltas[2:]), axis=(0, 1)))})

print("clock64 cycles (median): tmem ld -> topk, topk -> writes:", np.median(np.array(cyc[2:]), axis=0))
