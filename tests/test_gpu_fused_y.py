"""GEMM2 with the combine fused (FusedY, kernels/ffn_gemm.cu; default for top-2 on
one GPU on the 2-SM prefill kernel): no expert-output rows are written and no
combine kernel runs; of a token's two rows the first to finish an n tile parks
its bf16 output in y and the second writes the slot-order weighted sum — the
combine kernel's arithmetic.  Checked against the oracle (per-row 2e-2) and BIT
FOR BIT against the yp + combine-kernel path (MOE_FUSED_Y=0), whichever row
arrives first, over repeated / re-routed forwards and CUDA-graph replays (the
per-(token, n tile) counters reset themselves)."""
import os

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


def _layer(fused, E, k, d, ff, T, graphs=False, cap=0):
    os.environ["MOE_FUSED_Y"] = "1" if fused else "0"
    try:
        mem = 3.0 * d * ff * 2 / 1e6
        m = MoELayer(1, E, k, d, ff, max_tokens=T, cuda_graphs=graphs, expert_mem_mb=mem,
                     layer_mem_cap_mb=(E + cap) * mem)
    finally:
        del os.environ["MOE_FUSED_Y"]
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    return m, experts


@pytest.mark.parametrize("E,d,ff,T,cap", [
    (8, 1024, 512, 8192, 0),     # tcgen05 gate, three-kernel front, 2-SM K4 (mean rows 2048)
    (8, 1024, 512, 6000, 4),     # ragged m-tiles, straggler replicas (SYNC planning)
    (16, 2048, 256, 12000, 8),   # 16 experts (d = 2048: 8 GEMM2 n tiles per row)
])
def test_fused_y_vs_oracle_and_unfused(cuda, E, d, ff, T, cap):
    import torch
    k = 2
    x = wl.tokens(T, d, E, 1, 7)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    ys, errs = {}, {}
    for fused in (True, False):
        m, experts = _layer(fused, E, k, d, ff, T, cap=cap)
        outs = []
        for it in range(3):  # re-routed every forward: the arrival counters must reset themselves
            wg = wl.gate_weights(E, d, 1.2, 1, 0, it)
            m.set_gate(0, wg)
            yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            m.forward(0, xd, yd, MOE_PLAN_SYNC, it)
            torch.cuda.synchronize()
            y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
            outs.append(y)
            y_ref = oracle.layer_forward(x, wg, experts, [1] * E, k)[0]
            errs.setdefault(fused, []).append(row_rel_err(y, y_ref))
            assert errs[fused][-1] <= 2e-2, (fused, it, errs[fused][-1])
        if fused:  # run-to-run: the same bits whatever the arrival order
            wg = wl.gate_weights(E, d, 1.2, 1, 0, 2)
            m.set_gate(0, wg)
            yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            m.forward(0, xd, yd, MOE_PLAN_SYNC, 3)
            torch.cuda.synchronize()
            assert np.array_equal(oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16)), outs[2])
        ys[fused] = outs
        m.close()
    for it, (a, b) in enumerate(zip(ys[True], ys[False])):
        assert np.array_equal(a, b), (it, row_rel_err(a, b))

def test_fused_y_graph_replays(cuda):
    import torch
    E, k, d, ff, T = 8, 2, 1024, 512, 8192
    m, experts = _layer(True, E, k, d, ff, T, graphs=True)
    x = wl.tokens(T, d, E, 1, 3)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    gates = [wl.gate_weights(E, d, 1.2, 1, 0, it) for it in range(2)]
    gd = [torch.from_numpy(g.view(np.int16)).to(cuda) for g in gates]
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    first = {}
    for it in (0, 1, 0, 1, 0):
        m.set_gate_device(0, gd[it])
        m.forward(0, xd, yd, MOE_PLAN_FIXED, it)
        torch.cuda.synchronize()
        y = yd.cpu().numpy().copy()
        if it in first:
            assert np.array_equal(y, first[it]), it
        else:
            first[it] = y
            y_ref = oracle.layer_forward(x, gates[it], experts, [1] * E, k)[0]
            assert row_rel_err(oracle.bf16_to_f32(y.view(np.uint16)), y_ref) <= 2e-2
    m.close()
