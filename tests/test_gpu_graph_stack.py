"""Several layers' forwards recorded as ONE CUDA graph (moe_graph_begin /
moe_graph_end / moe_graph_launch): replays are bit-identical to the eager
forwards, re-read each layer's current gate weights (re-routing between
replays), and the last layer matches the oracle (ids bit-exact, per-row
relative error <= 2e-2).  Also the capture's error paths."""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer, MoeError
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu
TOL_ROW = 2e-2

CASES = [
    # E, k, d, ff, T, s, layers
    (64, 8, 2048, 1408, 256, 2.0, 3),  # cfg5 decode: fused front end + swap-AB K4 + L2 prefetch branch
    (8, 2, 1024, 3584, 2048, 1.2, 2),  # cfg1: fused front end (64 blocks) + 128-token swap tiles
    (8, 2, 1024, 512, 8192, 1.2, 2),   # prefill shape: tcgen05 gate + three-kernel front + 2-SM K4
]


def _rows_err(y, y_ref):
    den = np.maximum(np.max(np.abs(y_ref), axis=1), 1e-30)
    return float(np.max(np.max(np.abs(y - y_ref), axis=1) / den))


@pytest.mark.parametrize("E,k,d,ff,T,s,n_layers", CASES)
def test_graph_of_layers_matches_eager_and_oracle(cuda, E, k, d, ff, T, s, n_layers):
    import torch
    m = MoELayer(n_layers, E, k, d, ff, max_tokens=T)
    experts = [[wl.expert_weights(d, ff, 1, l, e) for e in range(E)] for l in range(n_layers)]
    for l in range(n_layers):
        for e in range(E):
            m.load_expert(l, e, *experts[l][e])
    xs = [wl.tokens(T, d, E, 1, 20 + l) for l in range(n_layers)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    gates = {(l, it): wl.gate_weights(E, d, s, 1, l, it) for l in range(n_layers) for it in (0, 1)}
    gd = {key: torch.from_numpy(g.view(np.int16)).to(cuda) for key, g in gates.items()}

    def eager(it):
        ys = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(n_layers)]
        for l in range(n_layers):
            m.set_gate_device(l, gd[(l, it)])
        for l in range(n_layers):
            m.forward(l, xd[l], ys[l], MOE_PLAN_FIXED, it)
        torch.cuda.synchronize()
        return [y.cpu().numpy().copy() for y in ys]

    ref = {it: eager(it) for it in (0, 1)}
    yg = [torch.full((T, d), 7, dtype=torch.int16, device=cuda) for _ in range(n_layers)]
    for l in range(n_layers):
        m.set_gate_device(l, gd[(l, 0)])
    m.graph_begin()
    for l in range(n_layers):
        m.forward(l, xd[l], yg[l], MOE_PLAN_FIXED, 0)
    gid = m.graph_end()
    torch.cuda.synchronize()
    assert all(int(torch.count_nonzero(y - 7)) == 0 for y in yg), "capture must not run the forwards"
    for it in (0, 1, 0):
        for l in range(n_layers):
            m.set_gate_device(l, gd[(l, it)])
        m.graph_launch(gid)
        torch.cuda.synchronize()
        for l in range(n_layers):
            assert np.array_equal(yg[l].cpu().numpy(), ref[it][l]), (it, l)
    # the last layer's routing / output vs the oracle (the ctx buffers hold the last forward's)
    l = n_layers - 1
    y_ref, ids_o, _, counts_o = oracle.layer_forward(xs[l], gates[(l, 0)], experts[l], [1] * E, k, round_h=True)
    assert np.array_equal(m.read_buffer(4, np.int32, (T, k)), ids_o)
    assert np.array_equal(m.read_buffer(7, np.int32, (E,)), counts_o)
    y = oracle.bf16_to_f32(yg[l].cpu().numpy().view(np.uint16))
    assert _rows_err(y, y_ref) <= TOL_ROW
    m.close()


def test_graph_capture_errors(cuda):
    import torch
    E, k, d, ff, T = 8, 2, 1024, 512, 64
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
    x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).to(cuda)
    y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    with pytest.raises((MoeError, ValueError)):
        m.graph_end()  # nothing open
    with pytest.raises((MoeError, ValueError)):
        m.graph_launch(0)  # unknown graph
    m.graph_begin()
    with pytest.raises((MoeError, ValueError)):
        m.graph_begin()  # already open
    with pytest.raises((MoeError, ValueError)):
        m.forward(0, x, y, MOE_PLAN_SYNC, 0, stats=True)  # stats inside a capture
    m.forward(0, x, y, MOE_PLAN_SYNC, 0)
    gid = m.graph_end()
    m.graph_launch(gid)
    m.forward(0, x, y, MOE_PLAN_FIXED, 1, stats=True)  # eager forwards still work after a capture
    torch.cuda.synchronize()
    m.close()


@pytest.mark.parametrize("T,mlp", [(256, False), (256, True), (8192, False)])
def test_graph_with_fused_predictor(cuda, T, mlp):
    """Layers whose gate kernel also scores the layer-aware predictor (K2: a
    linear slot, or an MLP slot) replay as one graph bit-identically to eager
    forwards, predictor histograms included (decode front end at T = 256, the
    tcgen05 prefill gate at T = 8192)."""
    import torch
    E, k, d, ff, n_layers = 16, 2, 1024, 256, 2
    rng = np.random.default_rng(5)
    m = MoELayer(n_layers, E, k, d, ff, max_tokens=T, num_predictor_targets=1)
    for l in range(n_layers):
        m.set_gate(l, wl.gate_weights(E, d, 1.2, 1, l, 0))
        wp = wl.gate_weights(E, d, 1.2, 1, 10 + l, 0)
        if mlp:
            m.set_predictor_mlp(l, 0, wp, rng.standard_normal((E, E)).astype(np.float32))
        else:
            m.set_predictor(l, 0, wp)
        for e in range(E):
            m.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 40 + l).view(np.int16)).to(cuda) for l in range(n_layers)]

    def run(graph):
        ys = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(n_layers)]
        if graph:
            m.graph_begin()
        for l in range(n_layers):
            m.forward(l, xd[l], ys[l], MOE_PLAN_FIXED, 0)
        if graph:
            m.graph_launch(m.graph_end())
        torch.cuda.synchronize()
        counts = m.read_buffer(7, np.int32, (2 * E,)).copy()  # the last layer's gate + predictor histograms
        return [y.cpu().numpy().copy() for y in ys], counts

    ye, ce = run(False)
    yg, cg = run(True)
    for l in range(n_layers):
        assert np.array_equal(ye[l], yg[l]), l
    assert np.array_equal(ce, cg)
    assert ce[E:].sum() == T * k  # the predictor slot's histogram covers every token
    m.close()
