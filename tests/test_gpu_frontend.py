"""The fused front end (kernels/frontend.cu: gate + top-k + plan +
dispatch in one cooperative launch) against the oracle and against the
three-kernel path it replaces (MOE_FRONTEND=0), bit for bit: ids, weights,
counts (gate and predictor histograms), row codes, the permuted rows, the
device plan and the layer output; eager and CUDA-graph replays."""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu
TOL_ROW = 2e-2


def _layer(monkeypatch, front, E, k, d, ff, T, npred, mlp, experts, wg, wps, w2s, graphs=False):
    monkeypatch.setenv("MOE_FRONTEND", "1" if front else "0")
    m = MoELayer(1, E, k, d, ff, max_tokens=T, num_predictor_targets=npred, cuda_graphs=graphs)
    m.set_gate(0, wg)
    for p, wp in enumerate(wps):
        if mlp and p == 0:
            m.set_predictor_mlp(0, p, wp, w2s)
        else:
            m.set_predictor(0, p, wp)
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    return m


def _forward(m, cuda, x, T, d, E, k, npred, it=0):
    import torch
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    m.forward(0, xd, yd, MOE_PLAN_FIXED, it)
    torch.cuda.synchronize()
    out = {
        "y": yd.cpu().numpy().copy(),
        "ids": m.read_buffer(4, np.int32, (T, k)),
        "wts": m.read_buffer(5, np.float32, (T, k)),
        "codes": m.read_buffer(6, np.uint32, (T, k)),
        "counts": m.read_buffer(7, np.int32, (E * (1 + npred),)),
        "xp": m.read_buffer(0, np.uint16, (T * k, d)),
    }
    out["plan"] = m.last_plan()
    return out


CASES = [
    # E, k, d, ff, T, s, npred, mlp
    (64, 8, 2048, 1408, 256, 2.0, 0, False),  # cfg5 decode, heavy skew
    (64, 8, 2048, 1408, 256, 1.2, 0, False),  # cfg5 at the milder skew
    (8, 2, 1024, 512, 1, 1.2, 0, False),      # one token
    (8, 2, 1024, 512, 33, 1.2, 1, False),     # ragged last block + linear predictor
    (16, 4, 2048, 256, 1000, 1.2, 2, True),   # 32 blocks (the limit), predictor MLP + linear slot
    (64, 8, 2048, 256, 77, 2.0, 1, False),    # 128 stacked logit columns, ragged
    (32, 6, 1024, 256, 500, 1.2, 0, False),   # k = 6
    (8, 2, 1024, 3584, 2048, 1.2, 0, False),  # cfg1: 64 blocks x 2 K splits
    (16, 2, 2048, 256, 4000, 1.2, 1, False),  # 125 blocks, no K split, predictor
]


@pytest.mark.parametrize("E,k,d,ff,T,s,npred,mlp", CASES)
def test_frontend_bitexact_vs_three_kernel_path_and_oracle(cuda, monkeypatch, E, k, d, ff, T, s, npred, mlp):
    rng = np.random.default_rng(T * 7 + E)
    wg = wl.gate_weights(E, d, s, 1, 0, 3)
    wps = [wl.gate_weights(E, d, s, 1, 1 + p, 3) for p in range(npred)]
    w2s = rng.standard_normal((E, E)).astype(np.float32) if mlp else None
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    x = wl.tokens(T, d, E, 1, 11)
    res = {}
    for front in (True, False):
        m = _layer(monkeypatch, front, E, k, d, ff, T, npred, mlp, experts, wg, wps, w2s)
        res[front] = _forward(m, cuda, x, T, d, E, k, npred)
        m.close()
    a, b = res[True], res[False]
    for key in ("ids", "wts", "codes", "counts", "y"):
        assert np.array_equal(a[key], b[key]), key
    assert np.array_equal(a["xp"], b["xp"])
    assert np.array_equal(a["plan"][0], b["plan"][0]) and np.array_equal(a["plan"][1], b["plan"][1])
    assert a["plan"][2] == b["plan"][2] == T * k
    # the oracle: routing, histograms and the stable permutation bit-exact
    ids_o, w_o, counts_o = oracle.gate(x, wg, k)
    assert np.array_equal(a["ids"], ids_o)
    assert np.array_equal(a["counts"][:E], counts_o)
    np.testing.assert_allclose(a["wts"], w_o, rtol=1e-5, atol=1e-6)
    for p, wp in enumerate(wps):
        want = oracle.predict_mlp(x, wp, w2s, k) if (mlp and p == 0) else oracle.gate(x, wp, k)[2]
        assert np.array_equal(a["counts"][E * (1 + p):E * (2 + p)], want), p
    (dg, dr), = oracle.dispatch([ids_o], k, E, np.ones(E, np.int32), np.zeros(E, np.int32))[0][:1]
    assert np.array_equal(a["codes"].reshape(-1).astype(np.int64), dr)
    # every permuted row is its token's row of x
    xr = x.view(np.uint16)
    tok = np.repeat(np.arange(T), k)
    assert np.array_equal(a["xp"][a["codes"].reshape(-1).astype(np.int64)], xr[tok])
    # output per token against the oracle (bf16 h rounding mirrored)
    idx = np.arange(T) if T <= 256 else np.sort(rng.choice(T, 256, replace=False))
    y = oracle.bf16_to_f32(a["y"].view(np.uint16))
    y_ref = oracle.layer_forward(x[idx], wg, experts, [1] * E, k, round_h=True)[0]
    scale = np.maximum(np.max(np.abs(y_ref), axis=1), 1e-6)
    err = np.max(np.abs(y[idx] - y_ref), axis=1) / scale
    assert float(err.max()) <= TOL_ROW


def test_frontend_graph_replay_rerouted(cuda, monkeypatch):
    """CUDA-graph replays of the fused front end, re-routed every step (new
    tokens through the same captured graph): outputs identical to eager."""
    import torch
    E, k, d, ff, T = 64, 8, 2048, 1408, 256
    wg = wl.gate_weights(E, d, 2.0, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    mg = _layer(monkeypatch, True, E, k, d, ff, T, 0, False, experts, wg, [], None, graphs=True)
    me = _layer(monkeypatch, True, E, k, d, ff, T, 0, False, experts, wg, [], None)
    xd = torch.empty((T, d), dtype=torch.int16, device=cuda)
    yg = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    ye = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    counts = []
    for it in range(4):
        x = wl.tokens(T, d, E, 1, 20 + it)
        xd.copy_(torch.from_numpy(x.view(np.int16)))
        torch.cuda.synchronize()  # the copy ran on torch's stream, the layer runs on the context's
        mg.forward(0, xd, yg, MOE_PLAN_FIXED, it)
        me.forward(0, xd, ye, MOE_PLAN_FIXED, it)
        torch.cuda.synchronize()
        assert torch.equal(yg, ye), it
        c = mg.read_buffer(7, np.int32, (E,))
        assert np.array_equal(c, oracle.gate(x, wg, k)[2]), it
        counts.append(c)
    assert any(not np.array_equal(counts[0], c) for c in counts[1:])  # the routing did change
    mg.close()
    me.close()
