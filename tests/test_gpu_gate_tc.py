"""The prefill gate on tcgen05 (gate_tc_kernel: 128-token tiles of x through a
TMA ring, M=128 x N<=32 UMMA into TMEM, per-thread top-k) against the oracle
and against the per-block mma.sync gate it replaces (MOE_GATE_TC=0): ids,
weights, gate and predictor histograms, row codes (which depend on the block
histograms) and the layer output, bit for bit."""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu


def _run(cuda, monkeypatch, tc, E, k, d, ff, T, npred, x, wg, wps, experts):
    import torch
    monkeypatch.setenv("MOE_GATE_TC", "1" if tc else "0")
    m = MoELayer(1, E, k, d, ff, max_tokens=T, num_predictor_targets=npred)
    m.set_gate(0, wg)
    for p, wp in enumerate(wps):
        m.set_predictor(0, p, wp)
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    m.forward(0, xd, yd, MOE_PLAN_FIXED, 0)
    torch.cuda.synchronize()
    out = dict(y=yd.cpu().numpy(), ids=m.read_buffer(4, np.int32, (T, k)), wts=m.read_buffer(5, np.float32, (T, k)),
               codes=m.read_buffer(6, np.uint32, (T, k)), counts=m.read_buffer(7, np.int32, (E * (1 + npred),)))
    m.close()
    return out


@pytest.mark.parametrize("E,k,d,ff,T,npred,s", [
    (8, 2, 4096, 256, 16384, 0, 1.2),   # cfg2 gate shape
    (8, 2, 4096, 256, 8193, 1, 1.2),    # ragged last tile and block, predictor (16 stacked rows)
    (16, 2, 4096, 256, 16384, 1, 1.2),  # cfg3 gate shape + predictor (32 stacked rows)
    (8, 4, 2048, 256, 20000, 3, 2.0),   # 4 stacked slots, top-4, heavy skew
    (4, 1, 1024, 256, 9000, 0, 1.2),    # top-1, N padded 4 -> 16
])
def test_tc_gate_bitexact(cuda, monkeypatch, E, k, d, ff, T, npred, s):
    wg = wl.gate_weights(E, d, s, 1, 0, 5)
    wps = [wl.gate_weights(E, d, s, 1, 1 + p, 5) for p in range(npred)]
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    x = wl.tokens(T, d, E, 1, 17)
    a = _run(cuda, monkeypatch, True, E, k, d, ff, T, npred, x, wg, wps, experts)
    b = _run(cuda, monkeypatch, False, E, k, d, ff, T, npred, x, wg, wps, experts)
    for key in ("ids", "wts", "counts", "codes", "y"):
        assert np.array_equal(a[key], b[key]), key
    ids_o, w_o, counts_o = oracle.gate(x, wg, k)
    assert np.array_equal(a["ids"], ids_o)
    assert np.array_equal(a["counts"][:E], counts_o)
    np.testing.assert_allclose(a["wts"], w_o, rtol=1e-5, atol=1e-6)
    for p, wp in enumerate(wps):
        assert np.array_equal(a["counts"][E * (1 + p):E * (2 + p)], oracle.gate(x, wp, k)[2]), p
