"""Gate kernels at the cfg5 decode shape through moe_gate_topk (no host
mirror) — compare their ncu durations with the forward's (mirrored) gate."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

E, k, d, T = 64, 8, 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = MoELayer(1, E, k, d, 1408, max_tokens=T)
m.set_gate(0, wl.gate_weights(E, d, 2.0, 1, 0, 0))
x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).cuda()
ids = torch.zeros((T, k), dtype=torch.int32, device="cuda")
w = torch.zeros((T, k), dtype=torch.float32, device="cuda")
c = torch.zeros(E, dtype=torch.int32, device="cuda")
for _ in range(6):
    m.gate(0, x, ids, w, c)
torch.cuda.synchronize()
m.close()
