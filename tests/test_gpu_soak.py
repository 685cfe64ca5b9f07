"""Many forwards through one context with varying token counts (0, 1, ragged,
max), two layers, SYNC and FIXED planning, CUDA-graph replay on and off: every
output stays within the oracle tolerance and the routing stays bit-exact —
catches state that leaks between calls (counters, rings, cached graphs/maps)."""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("graphs", [False, True])
def test_varying_batches_soak(cuda, graphs):
    import torch
    E, k, d, ff, Tmax, L = 8, 2, 1024, 1408, 384, 2
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(L, E, k, d, ff, max_tokens=Tmax, expert_mem_mb=mem, layer_mem_cap_mb=(E + 3) * mem,
                 cuda_graphs=graphs)
    experts = [[wl.expert_weights(d, ff, 1, l, e) for e in range(E)] for l in range(L)]
    for l in range(L):
        for e in range(E):
            m.load_expert(l, e, *experts[l][e])
    rng = np.random.default_rng(11)
    sizes = [0, 1, Tmax, 33, 257] + [int(v) for v in rng.integers(0, Tmax + 1, 25)]
    xbufs = {}
    for i, T in enumerate(sizes):
        l = i % L
        wg = wl.gate_weights(E, d, 1.4, 1, l, i)
        m.set_gate(l, wg)
        x = wl.tokens(T, d, E, 1, 300 + i) if T else np.zeros((0, d), np.uint16)
        # reuse device buffers per size so the graph cache is exercised
        key = (T, l)
        if key not in xbufs:
            xbufs[key] = (torch.empty((T, d), dtype=torch.int16, device=cuda),
                          torch.empty((T, d), dtype=torch.int16, device=cuda))
        xd, yd = xbufs[key]
        if T:
            xd.copy_(torch.from_numpy(x.view(np.int16)))
        mode = MOE_PLAN_SYNC if i % 3 else MOE_PLAN_FIXED
        m.forward(l, xd, yd, mode, i)
        m.sync()
        if T == 0:
            continue
        ids = m.read_buffer(4, np.int32, (T, k))
        y_ref, ids_o, _, _ = oracle.layer_forward(x, wg, experts[l], [1] * E, k, round_h=True)
        assert np.array_equal(ids, ids_o), (i, T)
        y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
        err = row_rel_err(y, y_ref)
        assert err <= 2e-2, (i, T, err)
    m.close()
