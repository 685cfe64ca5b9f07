"""An L-layer MoE stack driven the MoEless way (BASELINE.json cfg4).

Per (iteration, layer) — the reference's run() loop, simulator.cpp:113-262 —
the layer's gate (K1) and the fused predictor (K2, scoring layer l + d with
that layer's gate-shaped predictor weights) read the layer's
input once; the host planner then plans layer l + d from the PREDICTED loads
(scale_experts -> place_experts -> registry) while the GPU keeps running, and
layer l + d is evaluated on its actual loads, with measure_accuracy of the
prediction reported per layer (predictor.cpp:168-186).  Layers l < d have no
prediction and bootstrap from their load history (simulator.cpp:146-151).

Synthetic stand-ins (no checkpoint offline): every layer's gate carries its own
Zipf popularity permutation (workload.cpp:30-57); the predictor for layer l+d
is that layer's gate.  `forward` takes one input per layer: the tests give each
layer its own token batch (outputs checked per layer against the oracle), and
bench_configs.py cfg4 chains the layers through the residual stream
h_{l+1} = h_l + y_l, so layer l's predictor scores layer l+1 on the hidden
state that layer actually sees one residual update earlier — the accuracy it
reports measures that drift instead of comparing two iid Zipf draws.  All
layers share one set of random expert weights (loaded per layer).
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

from . import MOE_PLAN_PREDICTED, MoELayer
from . import workload as wl


class MoEStack:
    def __init__(self, num_layers: int, E: int, k: int, d: int, ff: int, tokens: int, extra_replicas: int,
                 zipf_s: float = 1.2, seed: int = 1, distance: int = 1, device: int = 0):
        mem = 3.0 * d * ff * 2 / 1e6
        self.L, self.E, self.k, self.d, self.T, self.distance = num_layers, E, k, d, tokens, distance
        self.layer = MoELayer(num_layers, E, k, d, ff, max_tokens=tokens, device=device, num_predictor_targets=1,
                              predictor_distance=distance, expert_mem_mb=mem,
                              layer_mem_cap_mb=extra_replicas * mem, keep_alive_iters=50)
        experts = [wl.expert_weights(d, ff, seed, 0, e) for e in range(E)]
        self.gates = [wl.gate_weights(E, d, zipf_s, seed, l, 0, num_layers=num_layers) for l in range(num_layers)]
        for l in range(num_layers):
            for e, w in enumerate(experts):
                self.layer.load_expert(l, e, *w)
            self.layer.set_gate(l, self.gates[l])
            if l + distance < num_layers:
                self.layer.set_predictor(l, 0, self.gates[l + distance])

    def forward(self, xs: List, ys: List, iteration: int, stats: bool = False, plan_mode: int = MOE_PLAN_PREDICTED):
        """Runs all layers back to back on the layer's stream; returns per-layer
        stats when requested (that synchronises after every layer)."""
        out = []
        for l in range(self.L):
            st = self.layer.forward(l, xs[l], ys[l], plan_mode, iteration, stats=stats)
            if stats:
                out.append(st)
        return out

    def close(self):
        self.layer.close()
