"""K2 (batched load predictor fused into the gate's read of x) and the
synchronous planner inside the forward, on the GPU against the oracle."""
import numpy as np
import pytest

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("E,k,d,T,npred", [(8, 2, 4096, 2048, 1), (8, 2, 1024, 777, 3), (16, 2, 2048, 512, 2),
                                           (64, 8, 2048, 256, 1), (8, 2, 4096, 6000, 1), (8, 2, 1024, 5000, 3)])
def test_predictor_counts_bitexact(cuda, E, k, d, T, npred):
    import torch
    m = MoELayer(1, E, k, d, 128, max_tokens=T, num_predictor_targets=npred)
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    wps = [wl.gate_weights(E, d, 1.2, 1, 1 + p, 0) for p in range(npred)]
    m.set_gate(0, wg)
    for p, wp in enumerate(wps):
        m.set_predictor(0, p, wp)
    x = wl.tokens(T, d, E, 1, 9)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    ids = torch.zeros((T, k), dtype=torch.int32, device=cuda)
    w = torch.zeros((T, k), dtype=torch.float32, device=cuda)
    counts = torch.zeros(E, dtype=torch.int32, device=cuda)
    pred = torch.zeros((npred, E), dtype=torch.int32, device=cuda)
    m.gate(0, xd, ids, w, counts, pred)
    torch.cuda.synchronize()
    ids_o, _, counts_o = oracle.gate(x, wg, k)
    assert np.array_equal(ids.cpu().numpy(), ids_o) and np.array_equal(counts.cpu().numpy(), counts_o)
    for p, wp in enumerate(wps):
        assert np.array_equal(pred[p].cpu().numpy(), oracle.gate(x, wp, k)[2])
    pred2 = torch.zeros((npred, E), dtype=torch.int32, device=cuda)
    m.predict_loads(0, xd, pred2)
    torch.cuda.synchronize()
    assert torch.equal(pred, pred2)
    # predictor accuracy metric (predictor.cpp:168-186) on the predicted vs actual loads
    acc = pk.measure_accuracy(pred[0].cpu().numpy(), counts.cpu().numpy())
    assert 0.0 <= acc <= 1.0
    m.close()


def test_sync_planner_inside_forward_matches_host_planner(cuda):
    import torch
    E, k, d, ff, T = 8, 2, 1024, 1408, 1024
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=4 * mem, keep_alive_iters=50)
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    m.set_gate(0, wg)
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    reg = pk.ReplicaRegistry(50)
    for it in range(3):
        x = wl.tokens(T, d, E, 1, it)
        xd = torch.from_numpy(x.view(np.int16)).to(cuda)
        yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
        st = m.forward(0, xd, yd, MOE_PLAN_SYNC, it, stats=True)
        counts = np.array(st.counts[:E])
        plan = pk.scale_experts(counts, mem, 4 * mem, 0.2)
        placed = pk.place_experts(plan, 1, 180000.0, reg, it)
        pk.update_registry(reg, plan.replica_counts, placed.flat(), 1, 0, it)
        assert st.replica_count == plan.total_replicas()
        assert (st.warm_count, st.cold_count) == (placed.warm_count, placed.cold_count)
        y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
        idx = np.arange(0, T, 37)
        y_ref = oracle.layer_forward(x[idx], wg, experts, [1] * E, k)[0]
        assert row_rel_err(y[idx], y_ref) <= 2e-2
    m.close()


def test_predicted_planning_distance_two(cuda):
    """MOE_PLAN_PREDICTED with predictor distance d = 2 over a 5-layer stack:
    layer l's fused predictor scores layer l + 2, layers 0-1 bootstrap from
    history (simulator.cpp:146-151), layers 2-4 run on placements planned two
    layers ahead; outputs equal the fixed-placement layer."""
    import torch
    from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_PREDICTED, MoELayer
    from paper_2603_06350_b200 import workload as wl
    L, E, k, d, ff, T, dist = 5, 8, 2, 1024, 1408, 256, 2
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(L, E, k, d, ff, max_tokens=T, num_predictor_targets=1, predictor_distance=dist,
                 expert_mem_mb=mem, layer_mem_cap_mb=(E + 3) * mem)
    ref = MoELayer(L, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    gates = [wl.gate_weights(E, d, 1.5, 1, l, 0) for l in range(L)]
    for mm in (m, ref):
        for l in range(L):
            mm.set_gate(l, gates[l])
            for e in range(E):
                mm.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    for l in range(L - dist):
        m.set_predictor(l, 0, gates[l + dist])
    xs = [torch.from_numpy(wl.tokens(T, d, E, 1, 40 + l).view(np.int16)).to(cuda) for l in range(L)]
    for it in range(3):
        sts = []
        for l in range(L):
            y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            sts.append(m.forward(l, xs[l], y, MOE_PLAN_PREDICTED, it, stats=True))
            y1 = torch.zeros_like(y)
            ref.forward(l, xs[l], y1, MOE_PLAN_FIXED, it)
            ref.sync()
            assert torch.equal(y, y1), (it, l)
        assert [st.plan_source for st in sts] == [3, 3, 2, 2, 2], [st.plan_source for st in sts]
        for st in sts[dist:]:
            assert 0.9 <= st.predictor_accuracy <= 1.0  # the predictor is layer l+2's own gate
    m.close()
    ref.close()


@pytest.mark.parametrize("E,k,d,T,npred,mlp_slots", [(8, 2, 4096, 2048, 1, (0,)), (16, 2, 1024, 777, 3, (0, 2)),
                                                     (64, 8, 2048, 300, 2, (1,)), (8, 2, 1024, 5000, 2, (0, 1))])
def test_predictor_mlp_counts_bitexact(cuda, E, k, d, T, npred, mlp_slots):
    """The batched predictor MLP (moe_set_predictor_mlp): hidden = relu of the
    slot's stacked rows, W2 (arbitrary fp32) applied per token in the gate
    kernel; histograms bit-identical to the oracle's fmaf chain, linear slots
    unchanged beside MLP slots, w2=None returns a slot to linear."""
    import torch
    rng = np.random.default_rng(E * 1000 + T)
    m = MoELayer(1, E, k, d, 128, max_tokens=T, num_predictor_targets=npred)
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    wps = [wl.gate_weights(E, d, 1.2, 1, 1 + p, 0) for p in range(npred)]
    w2s = {p: rng.standard_normal((E, E)).astype(np.float32) for p in mlp_slots}
    m.set_gate(0, wg)
    for p, wp in enumerate(wps):
        if p in w2s:
            m.set_predictor_mlp(0, p, wp, w2s[p])
        else:
            m.set_predictor(0, p, wp)
    x = wl.tokens(T, d, E, 1, 9)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    ids = torch.zeros((T, k), dtype=torch.int32, device=cuda)
    w = torch.zeros((T, k), dtype=torch.float32, device=cuda)
    counts = torch.zeros(E, dtype=torch.int32, device=cuda)
    pred = torch.zeros((npred, E), dtype=torch.int32, device=cuda)
    m.gate(0, xd, ids, w, counts, pred)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), oracle.gate(x, wg, k)[0])
    for p, wp in enumerate(wps):
        want = oracle.predict_mlp(x, wp, w2s[p], k) if p in w2s else oracle.gate(x, wp, k)[2]
        assert np.array_equal(pred[p].cpu().numpy(), want), p
    pred2 = torch.zeros_like(pred)
    m.predict_loads(0, xd, pred2)
    torch.cuda.synchronize()
    assert torch.equal(pred, pred2)
    p0 = mlp_slots[0]
    m.set_predictor_mlp(0, p0, None, None)  # back to linear, rows kept
    m.predict_loads(0, xd, pred2)
    torch.cuda.synchronize()
    assert np.array_equal(pred2[p0].cpu().numpy(), oracle.gate(x, wps[p0], k)[2])
    m.close()


def test_predictor_mlp_predicted_planning(cuda):
    """MOE_PLAN_PREDICTED driven by an MLP predictor (W2 = identity, so the
    scores are relu of layer l+1's gate logits): every layer after the first
    runs on the predicted placement and its output equals the fixed-placement
    layer's.  (The synthetic gate logits are mostly negative, so relu ties
    many scores at 0 and the accuracy is well below the linear predictor's.)"""
    import torch
    from paper_2603_06350_b200 import MOE_PLAN_FIXED, MOE_PLAN_PREDICTED
    L, E, k, d, ff, T = 3, 8, 2, 1024, 1408, 256
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(L, E, k, d, ff, max_tokens=T, num_predictor_targets=1, predictor_distance=1,
                 expert_mem_mb=mem, layer_mem_cap_mb=(E + 3) * mem)
    ref = MoELayer(L, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    gates = [wl.gate_weights(E, d, 1.5, 1, l, 0) for l in range(L)]
    for mm in (m, ref):
        for l in range(L):
            mm.set_gate(l, gates[l])
            for e in range(E):
                mm.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    for l in range(L - 1):
        m.set_predictor_mlp(l, 0, gates[l + 1], np.eye(E, dtype=np.float32))
    xs = [torch.from_numpy(wl.tokens(T, d, E, 1, 60 + l).view(np.int16)).to(cuda) for l in range(L)]
    for it in range(2):
        for l in range(L):
            y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            st = m.forward(l, xs[l], y, MOE_PLAN_PREDICTED, it, stats=True)
            y1 = torch.zeros_like(y)
            ref.forward(l, xs[l], y1, MOE_PLAN_FIXED, it)
            ref.sync()
            assert torch.equal(y, y1), (it, l)
            if l >= 1:
                assert st.plan_source == 2 and 0.0 <= st.predictor_accuracy <= 1.0
    m.close()
    ref.close()
