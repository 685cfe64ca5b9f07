"""Small layer forward for compute-sanitizer runs (memcheck / racecheck /
synccheck over K1 gate, K3 dispatch, K4 grouped GEMMs, K5 combine)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

E, k, d, ff, T = 8, 2, 256, 256, 200
m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=1.0, layer_mem_cap_mb=3.0)
m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).cuda()
y = torch.zeros((T, d), dtype=torch.int16, device="cuda")
for it in range(2):
    m.forward(0, x, y, MOE_PLAN_SYNC, it)
m.sync()
print("forward ok", float(y.float().abs().sum()))
