"""The CPU reference path of one MoE layer — BASELINE INFRASTRUCTURE ONLY.

Used by bench.py's reference arm (`--impl reference`) and its cpu_baseline
leg, never by the product.  One forward of the layer on the host:

  planner   the UNMODIFIED reference's per-layer path (oracle/_ref,
            ref_cpu_layer_path): route_tokens -> predict -> scale_experts ->
            place_experts -> layer_forward_time -> update_registry, exactly as
            run() sequences it (simulator.cpp:116-201), on the step's tokens;
  data      the oracle restatement of what the reference only models
            analytically (cost_model.cpp:91-122): gate GEMV + softmax + top-k
            (orc_gate, C/OpenMP), the stable integer dispatch (orc_dispatch),
            the SwiGLU expert FFN in fp32 on the host BLAS (OpenBLAS sgemm,
            all threads; weights resident as fp32, converted once like the
            GPU keeps its weights resident), and the weighted combine.

Every token's work is independent (per-token routing and FFN rows), so the
cost is linear in the tokens of a step; `forward` reports its own time.
"""
from __future__ import annotations

import time

import numpy as np

from . import P, bf16_to_f32, dispatch, gate, ref


class CpuLayer:
    def __init__(self, E, k, d, ff, experts, s=1.2, seed=1, extra_replicas=4):
        self.E, self.k, self.d, self.ff = E, k, d, ff
        self.s, self.seed = s, seed
        self.mem = 3.0 * d * ff * 2 / 1e6
        self.cap = extra_replicas * self.mem
        # resident fp32 weights in nn.Linear layout; sgemm reads them transposed
        self.w13 = [bf16_to_f32(np.concatenate([w1, w3])) for (w1, w3, _) in experts]
        self.w2 = [bf16_to_f32(w2) for (_, _, w2) in experts]
        self.ref = ref()

    def planner(self, tokens):
        """The reference's own per-layer CPU path (None when oracle/_ref is absent)."""
        if self.ref is None:
            return None
        loads = np.zeros(self.E, np.int64)
        dt = self.ref.ref_cpu_layer_path(tokens, self.E, self.k, self.s, self.seed, 1, self.mem, self.cap, 1,
                                         P(loads))
        return loads if dt >= 0 else None

    def forward(self, x, wg):
        """y [T, d] fp32 for bf16 tokens x [T, d] and gate wg [E, d]; returns (y, seconds)."""
        t0 = time.perf_counter()
        T = x.shape[0]
        self.planner(T)
        ids, w, counts = gate(x, wg, self.k)
        (_, rows), = dispatch([ids], self.k, self.E, [1] * self.E, [0] * self.E)[0][:1]
        rows = rows.reshape(T, self.k)
        xf = bf16_to_f32(x)
        Y = np.empty((T * self.k, self.d), np.float32)
        base = 0
        for e in range(self.E):
            n = int(counts[e])
            if n == 0:
                continue
            # the rows of expert e in dispatch order: row base + i <- (t, j)
            tj = np.nonzero((rows >= base) & (rows < base + n))
            order = np.argsort(rows[tj])
            xs = xf[tj[0][order]]
            gu = xs @ self.w13[e].T
            g, u = gu[:, :self.ff], gu[:, self.ff:]
            h = (g / (1.0 + np.exp(-g))) * u
            Y[base:base + n] = h @ self.w2[e].T
            base += n
        y = np.zeros((T, self.d), np.float32)
        for j in range(self.k):
            y += w[:, j:j + 1] * Y[rows[:, j]]
        return y, time.perf_counter() - t0
