"""Small forwards for compute-sanitizer runs over the round-2 paths:
  default  the fused decode front end (gate + top-k + plan + dispatch, one
           cooperative launch), swap-AB K4 with the side-stream L2 prefetch, combine
  frontpred  the same with a predictor MLP slot and a linear slot (64 stacked rows)
  gatetc   the tcgen05 prefill gate (T >= 8192) + side-stream histogram copy
  threek   MOE_FRONTEND=0: split-K gate + finish + dispatch (the three-kernel path)
  2sm      the 2-SM cta_group::2 K4 with claimed tiles (MOE_GEMM_VARIANT=2sm)
  ids      moe_layer_forward_ids (route_ids kernel instead of the gate)
  stream   the streaming prefill gate (MOE_GATE_STREAM=1, T >= 148 blocks)
  gatetcpred the tcgen05 gate with a linear predictor slot (tree top-k over the smem row)
  2smbig   the 2-SM K4 on 256-row tiles with staged epilogue stores (mean rows > 1024)
  graph    two forwards recorded as one CUDA graph (moe_graph_begin/end) and replayed
  fusedy   top-2 prefill on the 2-SM K4 with the combine fused into GEMM2 (> 148 blocks)
  python profiles/sanitize_forward_r02.py <scenario>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

scenario = sys.argv[1] if len(sys.argv) > 1 else "default"
E, k, d, ff, T = 8, 2, 256, 256, 200
if scenario == "2sm":
    os.environ["MOE_GEMM_VARIANT"] = "2sm"
    T = 600
if scenario == "stream":
    os.environ["MOE_GATE_STREAM"] = "1"
    d, T = 512, 148 * 32 + 17
if scenario in ("gatetc", "gatetcpred"):
    T = 8192 + 17
if scenario == "2smbig":
    d, ff, T = 512, 256, 4096 + 40
if scenario == "fusedy":
    d, ff, T = 512, 256, 8192 + 40
if scenario == "threek":
    os.environ["MOE_FRONTEND"] = "0"
npred = 2 if scenario == "frontpred" else (1 if scenario == "gatetcpred" else 0)
m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=1.0, layer_mem_cap_mb=3.0, num_predictor_targets=npred)
m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
if npred == 2:
    m.set_predictor_mlp(0, 0, wl.gate_weights(E, d, 1.2, 1, 1, 0),
                        np.random.default_rng(0).standard_normal((E, E)).astype(np.float32))
    m.set_predictor(0, 1, wl.gate_weights(E, d, 1.2, 1, 2, 0))
elif npred == 1:
    m.set_predictor(0, 0, wl.gate_weights(E, d, 1.2, 1, 1, 0))
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).cuda()
y = torch.zeros((T, d), dtype=torch.int16, device="cuda")
if scenario == "graph":
    m.graph_begin()
    m.forward(0, x, y, MOE_PLAN_SYNC, 0)
    m.forward(0, x, y, MOE_PLAN_SYNC, 1)
    gid = m.graph_end()
    m.graph_launch(gid)
    m.graph_launch(gid)
for it in range(2):
    if scenario == "ids":
        ids = torch.from_numpy(np.stack([np.arange(T) % E, (np.arange(T) + 3) % E], 1).astype(np.int32)).cuda()
        m.forward_ids(0, x, ids, y, None, MOE_PLAN_SYNC, it)
    else:
        m.forward(0, x, y, MOE_PLAN_SYNC, it)
m.sync()
print(scenario, "forward ok", float(y.float().abs().sum()))
