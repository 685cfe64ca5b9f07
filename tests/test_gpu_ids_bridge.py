"""The SURVEY §8 c3 bridge: the REFERENCE's routing drives the GPU data path.

`oracle.route_ids` replays the reference's route_tokens stream per token
(proj/src/workload.cpp:188-230); its histogram equals the compiled reference's
`route_tokens().loads` (committed in tests/golden/route_loads.json by
tests/golden/make_golden.py, and checked live when oracle/_ref is built).
Those ids enter the layer through moe_layer_forward_ids (K1 skipped), so
every GPU-side integer is pinned to the reference itself:

  * the counts the device histogram produces == reference loads;
  * the placement the context's SYNC planner chose on those counts == the
    compiled reference's scale_experts + place_experts on the same loads;
  * the device plan's per-expert totals == reference loads, and per (rank,
    expert) its segment rows == the reference loads cut by the integer replica
    rule floor(n/R) + [r < n mod R], at G = 1 and at G = 2/4
    peer-memory ranks sharing the B200;
  * row codes (the permutation) == oracle.dispatch on the same ids;
  * outputs: per-token relative error <= 2e-2 vs the oracle FFN + combine.
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoeError, MoELayer
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "route_loads.json")
CASES = {tuple(e["case"]): e["loads"] for e in json.load(open(GOLD))}
TOL_ROW = 2e-2


def ref_loads(case):
    """Reference route_tokens loads: live from oracle/_ref when built, else the golden."""
    T, layer, it, E, k, s, seed, drift = case
    ref = oracle.ref()
    if ref is not None:
        loads = np.zeros(E, np.int64)
        assert ref.ref_route_tokens(T, layer, it, E, 8, s, seed, k, drift, oracle.P(loads)) == 0
        assert loads.tolist() == CASES[case]  # golden and live reference agree
    return np.array(CASES[case], np.int64)


def ref_plan(loads, E, G, mem, cap_mb, cv=0.2):
    """The compiled reference's scale_experts + place_experts on `loads` (fresh registry)."""
    ref = oracle.ref()
    if ref is None:
        return None
    la = np.ascontiguousarray(loads, np.int64)
    rc = np.zeros(E, np.int32)
    alloc, steps = np.zeros(1), np.zeros(1, np.int32)
    assert ref.ref_scale_experts(oracle.P(la), E, 0, mem, cap_mb, cv, 0, oracle.P(rc), oracle.P(alloc),
                                 oracle.P(steps), None, 0, None, None) == 0
    reg = ref.ref_registry_new(50)
    gpu = np.zeros(int(rc.sum()), np.int32)
    warm, cold = np.zeros(1, np.int32), np.zeros(1, np.int32)
    assert ref.ref_place_experts(reg, oracle.P(la), oracle.P(rc), E, 0, mem, G, 180000.0, 0, 0, 0.0, 1.0,
                                 oracle.P(gpu), oracle.P(warm), oracle.P(cold)) == 0
    ref.ref_registry_free(reg)
    return rc, gpu


def split_rows(loads, rc, rg, G):
    """Expected rows per (rank, expert): the integer replica split of the loads."""
    out = np.zeros((G, len(loads)), np.int64)
    f = 0
    for e, n in enumerate(loads):
        R = int(rc[e])
        for r in range(R):
            out[rg[f], e] += n // R + (1 if r < n % R else 0)
            f += 1
    return out


def seg_rows(segs, E):
    out = np.zeros(E, np.int64)
    for _, rows, slot in segs:
        out[slot] += rows
    return out


def tokens_forward(x, ids, w, experts):
    """Oracle y_t = sum_j w_tj FFN_{ids_tj}(x_t) for the given tokens (fp32, slot order)."""
    T, k = ids.shape
    Y = np.zeros((T, k, x.shape[1]), np.float32)
    for e in np.unique(ids):
        t, j = np.nonzero(ids == e)
        Y[t, j] = oracle.expert_ffn(np.ascontiguousarray(x[t]), *experts[e], round_h=True, round_y=True)
    y = np.zeros((T, x.shape[1]), np.float32)
    for j in range(k):
        y = (y + w[:, j:j + 1] * Y[:, j]).astype(np.float32)
    return y


def row_rel_err(y, y_ref):
    scale = np.maximum(np.max(np.abs(y_ref), axis=1), 1e-6)
    return np.max(np.abs(y - y_ref), axis=1) / scale


# (route case, d, ff, extra replicas of memory cap, sampled tokens for the output check)
SINGLE = [
    ((2048, 0, 0, 8, 2, 1.2, 1, 0), 1024, 3584, 4, 2048),     # cfg1 shape
    ((16384, 1, 3, 8, 2, 1.2, 1, 0), 4096, 14336, 4, 1024),   # cfg2 Mixtral
    ((16384, 2, 5, 16, 2, 1.2, 1, 0), 4096, 6400, 8, 1024),   # cfg3 Phi-3.5 shape
    ((256, 0, 1, 64, 8, 1.2, 1, 0), 2048, 1408, 16, 256),     # cfg5 decode
    ((256, 3, 7, 64, 8, 2.0, 1, 0), 2048, 1408, 16, 256),     # cfg5 heavy skew
    ((1000, 1, 250, 8, 2, 1.2, 7, 100), 1024, 1408, 3, 1000),  # drifted popularity (period 100)
    ((50, 0, 0, 4, 4, 1.2, 1, 0), 256, 256, 2, 50),           # k == E
]


@pytest.mark.parametrize("case,d,ff,extra,sample", SINGLE)
def test_reference_routing_through_gpu_layer(cuda, case, d, ff, extra, sample):
    import torch
    T, layer, it, E, k, s, seed, drift = case
    if case not in CASES:
        pytest.skip("case has no golden")
    loads = ref_loads(case)
    ids, lo = oracle.route_ids(T, layer, it, E, s, seed, k, drift)
    assert np.array_equal(lo, loads) and np.array_equal(np.bincount(ids.reshape(-1), minlength=E), loads)
    rng = np.random.default_rng(T)
    w = rng.random((T, k)).astype(np.float32)
    w /= w.sum(axis=1, keepdims=True)
    x = wl.tokens(T, d, E, seed, it)
    experts = [wl.expert_weights(d, ff, seed, 0, e) for e in range(E)]
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=(E + extra) * mem)
    for e, wt in enumerate(experts):
        m.load_expert(0, e, *wt)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    idd = torch.from_numpy(ids).to(cuda)
    wd = torch.from_numpy(w).to(cuda)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    st = m.forward_ids(0, xd, idd, yd, wd, MOE_PLAN_SYNC, it, stats=True)
    torch.cuda.synchronize()
    # counts: the device histogram of the reference's ids == reference loads
    assert np.array_equal(np.array(st.counts[:E], np.int64), loads)
    # placement: the context's planner on those counts == the compiled reference's
    rc, rg = m.placement(0)
    want = ref_plan(loads, E, 1, mem, (E + extra) * mem)
    if want is not None:
        assert np.array_equal(rc, want[0]) and np.array_equal(rg, want[1])
    # the device plan: per-expert totals and segment rows == integer split of the loads
    n_e, segs, rows_local = m.last_plan()
    assert np.array_equal(n_e.astype(np.int64), loads)
    assert np.array_equal(seg_rows(segs, E), split_rows(loads, rc, rg, 1)[0])
    assert rows_local == T * k == st.rows_local
    # the permutation
    codes = m.read_buffer(6, np.uint32, (T, k)).astype(np.int64)
    (dg, dr), = oracle.dispatch([ids], k, E, rc, rg)[0][:1]
    assert np.array_equal(codes.reshape(-1), dr)
    # outputs on sampled tokens
    idx = np.sort(rng.choice(T, size=min(sample, T), replace=False))
    y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))[idx]
    y_ref = tokens_forward(x[idx], ids[idx], w[idx], experts)
    err = row_rel_err(y, y_ref)
    assert float(err.max()) <= TOL_ROW, float(err.max())
    m.close()


def test_empty_batch_through_ids_entry(cuda):
    import torch
    E, k, d, ff = 8, 2, 256, 256
    m = MoELayer(1, E, k, d, ff, max_tokens=16)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    x = torch.zeros((1, d), dtype=torch.int16, device=cuda)[:0]
    ids = torch.zeros((1, k), dtype=torch.int32, device=cuda)[:0]
    y = torch.zeros((1, d), dtype=torch.int16, device=cuda)[:0]
    st = m.forward_ids(0, x, ids, y, None, MOE_PLAN_SYNC, 0, stats=True)
    assert list(st.counts[:E]) == [0] * E and st.rows_local == 0
    m.close()


@pytest.mark.parametrize("bad", ["range", "repeat", "negative"])
def test_invalid_ids_raise_einval(cuda, bad):
    import torch
    E, k, d, ff, T = 8, 2, 256, 256, 40
    m = MoELayer(1, E, k, d, ff, max_tokens=T)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    ids = np.tile(np.array([[0, 1]], np.int32), (T, 1))
    ids[33] = {"range": [3, 8], "repeat": [5, 5], "negative": [-1, 2]}[bad]
    x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).to(cuda)
    y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    with pytest.raises(ValueError, match="token 33"):
        m.forward_ids(0, x, torch.from_numpy(ids).to(cuda), y, None, MOE_PLAN_FIXED, 0, stats=True)
    # the context stays usable and a valid call succeeds
    ids[33] = [2, 3]
    st = m.forward_ids(0, x, torch.from_numpy(ids).to(cuda), y, None, MOE_PLAN_FIXED, 1, stats=True)
    assert st.counts[0] == T - 1 and st.counts[2] == 1
    m.close()


@pytest.mark.parametrize("G,case,d,ff,extra", [
    (2, (2048, 0, 0, 8, 2, 1.2, 1, 0), 1024, 1408, 4),
    (4, (256, 0, 1, 64, 8, 1.2, 1, 0), 2048, 1408, 16),
    (4, (256, 3, 7, 64, 8, 2.0, 1, 0), 2048, 1408, 16),
])
def test_reference_routing_expert_parallel(cuda, G, case, d, ff, extra):
    """G peer-memory ranks share the B200; the reference's T tokens are sharded
    contiguously over the ranks (global order = (rank, token) = reference token
    order).  Every rank plans the same placement from the all-gathered
    histogram; per (rank, expert) the received rows are the integer split."""
    import torch
    T, layer, it, E, k, s, seed, drift = case
    loads = ref_loads(case)
    ids, _ = oracle.route_ids(T, layer, it, E, s, seed, k, drift)
    bounds = [T * r // G for r in range(G + 1)]
    x = wl.tokens(T, d, E, seed, it)
    experts = [wl.expert_weights(d, ff, seed, 0, e) for e in range(E)]
    mem = 3.0 * d * ff * 2 / 1e6
    Tmax = max(bounds[r + 1] - bounds[r] for r in range(G))
    ms = [MoELayer(1, E, k, d, ff, max_tokens=Tmax, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   expert_mem_mb=mem, layer_mem_cap_mb=(E + extra) * mem) for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
        for e, wt in enumerate(experts):
            m.load_expert(0, e, *wt)
    xs = [torch.from_numpy(np.ascontiguousarray(x[bounds[r]:bounds[r + 1]]).view(np.int16)).to(cuda)
          for r in range(G)]
    ids_r = [np.ascontiguousarray(ids[bounds[r]:bounds[r + 1]]) for r in range(G)]
    idd = [torch.from_numpy(a).to(cuda) for a in ids_r]
    ys = [torch.zeros((bounds[r + 1] - bounds[r], d), dtype=torch.int16, device=cuda) for r in range(G)]
    with ThreadPoolExecutor(G) as ex:
        sts = list(ex.map(lambda r: ms[r].forward_ids(0, xs[r], idd[r], ys[r], None, MOE_PLAN_SYNC, it,
                                                     stats=True), range(G)))
    torch.cuda.synchronize()
    rc, rg = ms[0].placement(0)
    for m in ms[1:]:
        rc2, rg2 = m.placement(0)
        assert np.array_equal(rc, rc2) and np.array_equal(rg, rg2)  # identical decisions
    want = ref_plan(loads, E, G, mem, (E + extra) * mem)
    if want is not None:
        assert np.array_equal(rc, want[0]) and np.array_equal(rg, want[1])
    expect = split_rows(loads, rc, rg, G)
    per_rank = oracle.dispatch(ids_r, k, E, rc, rg)[0]
    for r, m in enumerate(ms):
        assert np.array_equal(np.array(sts[r].counts[:E]), np.bincount(ids_r[r].reshape(-1), minlength=E))
        n_e, segs, rows_local = m.last_plan()
        assert np.array_equal(n_e.astype(np.int64), loads)  # global totals on every rank
        assert np.array_equal(seg_rows(segs, E), expect[r])
        assert rows_local == int(expect[r].sum())
        codes = m.read_buffer(6, np.uint32, ids_r[r].shape).astype(np.int64).reshape(-1)
        dg, dr = per_rank[r]
        assert np.array_equal(codes >> 28, dg) and np.array_equal(codes & ((1 << 28) - 1), dr)
    # outputs: every rank's tokens vs the oracle (equal weights 1/k)
    for r in range(G):
        n = bounds[r + 1] - bounds[r]
        w = np.full((n, k), 1.0 / k, np.float32)
        y = oracle.bf16_to_f32(ys[r].cpu().numpy().view(np.uint16))
        y_ref = tokens_forward(x[bounds[r]:bounds[r + 1]], ids_r[r], w, experts)
        assert float(row_rel_err(y, y_ref).max()) <= TOL_ROW
    for m in ms:
        m.close()
