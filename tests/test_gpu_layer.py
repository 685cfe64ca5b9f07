"""GPU parity: the sm_100a data path (via the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star): routing ids, load counts and permutations
bit-exact; FFN/combine outputs within max relative error 2e-2 (bf16 inputs,
fp32 accumulate vs the fp32 oracle), measured as
    max|y_gpu - y_ref| / max|y_ref|  <= 2e-2
and, against the oracle that mirrors the device's bf16 rounding of h and Y,
a much tighter 1e-2 bound per element relative to the row scale.
"""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer, exchange_plan
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu

TOL_REL = 2e-2


def _to_dev(a, torch):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def _build(E, k, d, ff, T, seed=1, layer=0, iteration=0, s=1.2):
    x = wl.tokens(T, d, E, seed, iteration)
    wg = wl.gate_weights(E, d, s, seed, layer, iteration)
    experts = [wl.expert_weights(d, ff, seed, layer, e) for e in range(E)]
    return x, wg, experts


@pytest.mark.parametrize("E,k,d,T", [(8, 2, 1024, 2048), (16, 2, 4096, 1024), (64, 8, 2048, 256),
                                     (8, 2, 4096, 999), (64, 8, 2048, 1),
                                     # >= 4736 tokens: the TMA-staged gate kernel (ragged last block)
                                     (8, 2, 4096, 5001), (16, 2, 1024, 8192), (32, 4, 2048, 4800)])
def test_gate_ids_counts_bitexact(cuda, E, k, d, T):
    import torch
    x, wg, _ = _build(E, k, d, 128, T)
    ids_o, w_o, counts_o = oracle.gate(x, wg, k)
    m = MoELayer(1, E, k, d, 128, max_tokens=T)
    m.set_gate(0, wg)
    xd = _to_dev(x, torch)
    ids = torch.zeros((T, k), dtype=torch.int32, device=cuda)
    w = torch.zeros((T, k), dtype=torch.float32, device=cuda)
    counts = torch.zeros(E, dtype=torch.int32, device=cuda)
    m.gate(0, xd, ids, w, counts)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), ids_o)
    assert np.array_equal(counts.cpu().numpy(), counts_o)
    assert int(counts.sum()) == T * k
    np.testing.assert_allclose(w.cpu().numpy(), w_o, rtol=1e-5, atol=1e-6)
    m.close()


def _layer_case(cuda, E, k, d, ff, T, rc, seed=3):
    import torch
    x, wg, experts = _build(E, k, d, ff, T, seed=seed)
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    m.set_gate(0, wg)
    for e, (w1, w3, w2) in enumerate(experts):
        m.load_expert(0, e, w1, w3, w2)
    R = int(np.sum(rc))
    m.set_placement(0, rc, [0] * R)
    xd = _to_dev(x, torch)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    st = m.forward(0, xd, yd, MOE_PLAN_FIXED, 0, stats=True)
    torch.cuda.synchronize()
    y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
    y_ref, ids_o, w_o, counts_o = oracle.layer_forward(x, wg, experts, rc, k, round_h=True)
    # routing and permutation: bit-exact against the oracle's dispatch
    ids = m.read_buffer(4, np.int32, (T, k))
    codes = m.read_buffer(6, np.uint32, (T, k))
    assert np.array_equal(ids, ids_o)
    (dg, dr), = oracle.dispatch([ids_o], k, E, rc, [0] * R)[0][:1]
    assert np.array_equal(codes.reshape(-1).astype(np.int64), dr)
    return m, st, y, y_ref, ids_o, counts_o


def _rel_err(y, y_ref):
    return row_rel_err(y, y_ref)


@pytest.mark.parametrize("E,k,d,ff,T,rc", [
    (8, 2, 1024, 3584, 512, [1] * 8),
    (8, 2, 1024, 3584, 384, [2, 1, 3, 1, 1, 1, 1, 2]),
    (16, 2, 1024, 1408, 300, [1] * 16),
    (64, 8, 2048, 1408, 64, [1] * 60 + [2, 3, 1, 2]),
])
def test_layer_forward_vs_oracle(cuda, E, k, d, ff, T, rc):
    m, st, y, y_ref, ids_o, counts_o = _layer_case(cuda, E, k, d, ff, T, rc)
    assert np.array_equal(np.array(st.counts[:E]), counts_o)
    err = _rel_err(y, y_ref)
    assert err <= TOL_REL, err
    # per-row check against the bf16-mirroring oracle
    scale = np.maximum(np.max(np.abs(y_ref), axis=1, keepdims=True), 1e-6)
    assert float(np.max(np.abs(y - y_ref) / scale)) <= 2e-2
    # every routed row was computed exactly once
    assert st.rows_local == T * k
    m.close()


def test_layer_forward_matches_torch_fp32(cuda):
    """Independent fp32 reference built with torch (not the oracle)."""
    import torch
    E, k, d, ff, T = 8, 2, 1024, 3584, 256
    x, wg, experts = _build(E, k, d, ff, T, seed=11)
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    m.set_gate(0, wg)
    for e, (w1, w3, w2) in enumerate(experts):
        m.load_expert(0, e, w1, w3, w2)
    xd = _to_dev(x, torch)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    m.forward(0, xd, yd)
    torch.cuda.synchronize()
    y = torch.from_numpy(oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16)))
    f = lambda a: torch.from_numpy(oracle.bf16_to_f32(a))
    xf, wgf = f(x), f(wg)
    logits = xf @ wgf.T
    probs = torch.softmax(logits, dim=-1)
    topv, topi = torch.topk(probs, k, dim=-1)
    topv = topv / topv.sum(-1, keepdim=True)
    ref = torch.zeros((T, d))
    for e, (w1, w3, w2) in enumerate(experts):
        rows, slot = torch.nonzero(topi == e, as_tuple=True)
        if len(rows) == 0:
            continue
        h = torch.nn.functional.silu(xf[rows] @ f(w1).T) * (xf[rows] @ f(w3).T)
        ref.index_add_(0, rows, topv[rows, slot, None] * (h @ f(w2).T))
    err = float((y - ref).abs().max() / ref.abs().max())
    assert err <= TOL_REL, err
    m.close()


@pytest.mark.parametrize("E,k,d,ff,T,rc", [
    (8, 2, 1024, 3584, 999, [2, 1, 3, 1, 1, 1, 1, 2]),
    (64, 8, 2048, 1408, 256, [1] * 60 + [2, 3, 1, 2]),
    (16, 2, 4096, 1408, 1, [1] * 16),
])
def test_gathered_gemm1_matches_dispatch_copy(cuda, monkeypatch, E, k, d, ff, T, rc):
    """Single GPU: GEMM1 gathering its rows from x with TMA gather4 (default)
    must give bit-identical outputs to GEMM1 over the dispatch kernel's
    permuted copy (MOE_GATHER=0), and the row -> token list it reads must be
    the inverse of the row codes."""
    import torch
    outs = []
    monkeypatch.setenv("MOE_GEMM_VARIANT", "1sm")  # gather is a 128-row-tile feature (decode shapes pick swap-AB)
    for flag in ("1", "0"):
        monkeypatch.setenv("MOE_GATHER", flag)
        m, st, y, y_ref, ids_o, counts_o = _layer_case(cuda, E, k, d, ff, T, rc)
        assert _rel_err(y, y_ref) <= TOL_REL
        if flag == "1":
            codes = m.read_buffer(6, np.uint32, (T, k)).reshape(-1).astype(np.int64)
            perm = m.read_buffer(11, np.int32, (T * k,))
            assert np.array_equal(np.sort(codes), np.arange(T * k))
            assert np.array_equal(perm[codes], np.repeat(np.arange(T), k))
        outs.append(y)
        m.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("E,k,d,ff,T,rc", [
    (8, 2, 1024, 3584, 999, [2, 1, 3, 1, 1, 1, 1, 2]),
    (64, 8, 2048, 1408, 256, [1] * 60 + [2, 3, 1, 2]),
    (16, 2, 4096, 1408, 1, [1] * 16),
    (8, 1, 1024, 1408, 300, [1] * 8),
])
def test_fused_combine_matches_combine_kernel(cuda, monkeypatch, E, k, d, ff, T, rc):
    """Single GPU: the combine fused into GEMM2's epilogue (MOE_FUSED_COMBINE=1; the last of a
    token's k rows per n tile sums them in slot order) must be bit-identical to
    the separate combine kernel (MOE_FUSED_COMBINE=0), on repeated forwards
    (the arrival counters reset themselves)."""
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("MOE_FUSED_COMBINE", flag)
        m, st, y, y_ref, ids_o, counts_o = _layer_case(cuda, E, k, d, ff, T, rc)
        assert _rel_err(y, y_ref) <= TOL_REL
        outs.append(y)
        m.close()
    assert np.array_equal(outs[0], outs[1])


def test_empty_batch_forward(cuda):
    """T = 0 (a rank or a step with no tokens): every kernel is skipped or
    degenerate, the call succeeds, nothing is routed, and the next non-empty
    forward is unaffected."""
    import torch
    E, k, d, ff = 8, 2, 1024, 1408
    x, wg, experts = _build(E, k, d, ff, 64, seed=5)
    m = MoELayer(1, E, k, d, ff, max_tokens=64)
    m.set_gate(0, wg)
    for e, (w1, w3, w2) in enumerate(experts):
        m.load_expert(0, e, w1, w3, w2)
    empty = torch.zeros((0, d), dtype=torch.int16, device=cuda)
    st = m.forward(0, empty, torch.zeros((0, d), dtype=torch.int16, device=cuda), MOE_PLAN_FIXED, 0, stats=True)
    assert st.rows_local == 0 and sum(st.counts[:E]) == 0
    xd = _to_dev(x, torch)
    yd = torch.zeros((64, d), dtype=torch.int16, device=cuda)
    m.forward(0, xd, yd, MOE_PLAN_FIXED, 1)
    torch.cuda.synchronize()
    y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
    y_ref = oracle.layer_forward(x, wg, experts, [1] * E, k, round_h=True)[0]
    assert _rel_err(y, y_ref) <= TOL_REL
    m.close()


def test_gate_exact_ties_pick_lower_expert(cuda):
    """Experts 2 and 5 (and 6, 7) get identical gate rows: their logits tie
    exactly for every token, and the top-k takes the LOWER index first, as the
    oracle does (route_tokens has no ties; this is the Mixtral-convention rule
    of DESIGN.md §K1)."""
    import torch
    E, k, d, T = 8, 2, 1024, 512
    x, wg, _ = _build(E, k, d, 128, T, seed=9)
    wg = wg.copy()
    wg[5] = wg[2]
    wg[7] = wg[6]
    ids_o, w_o, counts_o = oracle.gate(x, wg, k)
    m = MoELayer(1, E, k, d, 128, max_tokens=T)
    m.set_gate(0, wg)
    ids = torch.zeros((T, k), dtype=torch.int32, device=cuda)
    w = torch.zeros((T, k), dtype=torch.float32, device=cuda)
    counts = torch.zeros(E, dtype=torch.int32, device=cuda)
    m.gate(0, _to_dev(x, torch), ids, w, counts)
    torch.cuda.synchronize()
    ids = ids.cpu().numpy()
    assert np.array_equal(ids, ids_o)
    # an upper twin is only ever chosen right after its lower twin (equal logit)
    for lo, hi in ((2, 5), (6, 7)):
        rows, slot = np.nonzero(ids == hi)
        assert np.all(slot == 1) and np.all(ids[rows, 0] == lo)
        assert np.all(ids[ids[:, 0] == lo, 1] == hi)  # when the lower twin leads, the upper one follows
    m.close()


def test_device_gate_update_matches_host_upload(cuda):
    """moe_set_gate_weights_device (stream-ordered D2D copy of a resident gate)
    routes exactly like the host upload, call after call."""
    import torch
    E, k, d, ff, T = 8, 2, 1024, 1408, 256
    x, _, experts = _build(E, k, d, ff, T, seed=21)
    gates = [wl.gate_weights(E, d, 1.3, 1, 0, it) for it in range(3)]
    outs = []
    for dev in (False, True):
        m = MoELayer(1, E, k, d, ff, max_tokens=T)
        for e, (w1, w3, w2) in enumerate(experts):
            m.load_expert(0, e, w1, w3, w2)
        xd = _to_dev(x, torch)
        gd = torch.from_numpy(np.stack(gates).view(np.int16)).to(cuda)
        ys = []
        for it in range(3):
            if dev:
                m.set_gate_device(0, gd[it])
            else:
                m.set_gate(0, gates[it])
            yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            m.forward(0, xd, yd, MOE_PLAN_FIXED, it)
            ys.append(yd)
        m.sync()
        outs.append([y.cpu().numpy() for y in ys])
        m.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_forward_on_caller_stream_sees_uploads(cuda):
    """Gate / placement uploads go on the context's stream; a forward on a
    caller stream issued right after them must see them (and a later upload
    must not overtake the forward)."""
    import torch
    E, k, d, ff, T = 8, 2, 1024, 1408, 512
    x, wg, experts = _build(E, k, d, ff, T, seed=21)
    wg2 = wl.gate_weights(E, d, 2.0, 21, 0, 9)
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    ref = MoELayer(1, E, k, d, ff, max_tokens=T)
    for mm in (m, ref):
        for e, (w1, w3, w2) in enumerate(experts):
            mm.load_expert(0, e, w1, w3, w2)
    xd = _to_dev(x, torch)
    side = torch.cuda.Stream()
    outs = []
    for it, (g, rc) in enumerate([(wg, [1] * E), (wg2, [2, 1, 1, 1, 3, 1, 1, 1]), (wg, [1] * E)]):
        m.set_gate(0, g)
        m.set_placement(0, rc, [0] * sum(rc))
        y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
        m.forward(0, xd, y, MOE_PLAN_FIXED, it, stream=side.cuda_stream)
        outs.append(y)
    torch.cuda.synchronize()
    for g, y in zip((wg, wg2, wg), outs):
        ref.set_gate(0, g)
        y1 = torch.zeros_like(y)
        ref.forward(0, xd, y1)
        ref.sync()
        assert torch.equal(y, y1)
    m.close()
    ref.close()


def test_empty_forward_then_full(cuda):
    """T = 0 launches no dispatch; the next forward must not see a stale plan."""
    import torch
    E, k, d, ff, T = 8, 2, 1024, 1408, 300
    x, wg, experts = _build(E, k, d, ff, T, seed=22)
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    m.set_gate(0, wg)
    for e, (w1, w3, w2) in enumerate(experts):
        m.load_expert(0, e, w1, w3, w2)
    xd = _to_dev(x, torch)
    ys = []
    for t in (T, 0, T, 0, 0, T):
        y = torch.zeros((max(t, 1), d), dtype=torch.int16, device=cuda)[:t]
        m.forward(0, xd[:t], y, MOE_PLAN_FIXED, 0)  # eager, no timing events: PDL chain intact
        ys.append(y)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[2]) and torch.equal(ys[0], ys[5])
    m.close()
