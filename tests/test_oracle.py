"""The CPU oracle, pinned before it is trusted (CPU only).

* route replay vs the REFERENCE's route_tokens (committed goldens produced by
  the compiled, unmodified reference, and live against oracle/_ref when built);
* the reference's own workload tests restated (test_workload.cpp:161-201);
* gate / dispatch / FFN / combine against the committed golden fixtures and
  against independent numpy restatements.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


@pytest.mark.parametrize("entry", json.load(open(os.path.join(GOLD, "route_loads.json"))))
def test_route_replay_matches_reference_golden(entry):
    T, layer, it, E, k, s, seed, drift = entry["case"]
    ids, loads = oracle.route_ids(T, layer, it, E, s, seed, k, drift)
    assert loads.tolist() == entry["loads"]
    assert np.bincount(ids.reshape(-1), minlength=E).tolist() == entry["loads"]
    for row in ids:
        assert len(set(row.tolist())) == k  # distinct experts (workload.cpp:221-226)


def test_route_replay_matches_live_reference():
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(0)
    for _ in range(40):
        E = int(rng.integers(1, 70))
        k = int(rng.integers(1, min(E, 8) + 1))
        T = int(rng.integers(0, 3000))
        s = float(rng.choice([0.0, 0.8, 1.2, 2.0]))
        layer, it, seed = int(rng.integers(0, 8)), int(rng.integers(0, 1000)), int(rng.integers(0, 1 << 62))
        drift = int(rng.choice([0, 0, 50]))
        loads = np.zeros(E, np.int64)
        assert ref.ref_route_tokens(T, layer, it, E, 8, s, seed, k, drift, oracle.P(loads)) == 0
        _, lo = oracle.route_ids(T, layer, it, E, s, seed, k, drift)
        assert np.array_equal(lo, loads)


def test_popularity_matches_reference():
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference library not built")
    for E, layer, it, drift in [(8, 0, 0, 0), (16, 3, 5, 0), (64, 1, 250, 100), (8, 0, 99, 100)]:
        pr = np.zeros(E, np.int32)
        wr = np.zeros(E)
        assert ref.ref_popularity_perm(E, 4, 1.2, 1, layer, it, drift, oracle.P(pr), oracle.P(wr)) == 0
        po, wo = oracle.popularity(E, 1.2, 1, layer, it, drift)
        assert np.array_equal(pr, po)
        assert np.array_equal(wr, wo)


# reference test_workload.cpp:161-201 restated on the oracle
def test_route_conservation_and_keying():
    _, a = oracle.route_ids(400, 0, 3, 16, 1.2, 99, 2)
    assert a.sum() == 800 and (a >= 0).all()
    _, b = oracle.route_ids(400, 0, 3, 16, 1.2, 99, 2)
    assert np.array_equal(a, b)
    _, c = oracle.route_ids(400, 1, 3, 16, 1.2, 99, 2)
    _, d = oracle.route_ids(400, 0, 4, 16, 1.2, 99, 2)
    assert not np.array_equal(a, c) and not np.array_equal(a, d)


def test_route_topk_equal_experts_saturates():
    _, loads = oracle.route_ids(50, 0, 0, 4, 1.2, 1, 4)
    assert loads.tolist() == [50, 50, 50, 50]


def test_route_skew_band():
    perm, _ = oracle.popularity(16, 1.2, 21, 0)
    _, loads = oracle.route_ids(20000, 0, 0, 16, 1.2, 21, 1)
    frac = loads[perm[0]] / loads.sum()
    assert 0.30 < frac < 0.43


def test_gate_golden_and_exactness():
    g = load("gate_small.npz")
    ids, w, counts, logits = oracle.gate(g["x"], g["wg"], 2, want_logits=True)
    assert np.array_equal(ids, g["ids"]) and np.array_equal(counts, g["counts"])
    np.testing.assert_array_equal(w, g["w"])
    # logits on the synthetic grid are exact: float64 numpy gives the same values
    xf, wf = oracle.bf16_to_f32(g["x"]).astype(np.float64), oracle.bf16_to_f32(g["wg"]).astype(np.float64)
    np.testing.assert_array_equal(logits.astype(np.float64), xf @ wf.T)
    # top-k with lowest-index ties, softmax over the chosen k
    lg = xf @ wf.T
    for t in range(lg.shape[0]):
        order = sorted(range(lg.shape[1]), key=lambda e: (-lg[t, e], e))[:2]
        assert ids[t].tolist() == order
        p = np.exp(lg[t, order] - lg[t, order[0]])
        np.testing.assert_allclose(w[t], p / p.sum(), rtol=1e-6)
    assert counts.sum() == 2 * g["x"].shape[0]


def test_gate_ties_prefer_lowest_index():
    d, E = 16, 4
    x = oracle.f32_to_bf16(np.ones((3, d), np.float32))
    wg = oracle.f32_to_bf16(np.zeros((E, d), np.float32))
    ids, w, counts = oracle.gate(x, wg, 2)
    assert ids.tolist() == [[0, 1]] * 3 and counts.tolist() == [3, 3, 0, 0]
    np.testing.assert_allclose(w, 0.5)


def test_dispatch_golden():
    g = load("dispatch_small.npz")
    per, ss, sr, rows = oracle.dispatch([g["ids0"], g["ids1"]], 2, 8, g["rc"], g["rg"])
    assert np.array_equal(per[0][0], g["dg0"]) and np.array_equal(per[0][1], g["dr0"])
    assert np.array_equal(per[1][0], g["dg1"]) and np.array_equal(per[1][1], g["dr1"])
    assert np.array_equal(ss, g["seg_start"]) and np.array_equal(sr, g["seg_rows"])
    assert np.array_equal(rows, g["rows"])


def test_dispatch_rule_properties():
    """Integer even split (cost_model.cpp:98-106 made integer): replica sizes
    differ by at most one, larger ones first; every gpu's rows form a
    permutation of its segments; order inside a segment is (rank, token)."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        G, E, k = int(rng.integers(1, 5)), int(rng.integers(2, 12)), 2
        ids = []
        for _ in range(G):
            T = int(rng.integers(0, 80))
            ids.append(np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
                       if T else np.zeros((0, k), np.int32))
        rc = rng.integers(1, 4, E).astype(np.int32)
        rg = rng.integers(0, G, int(rc.sum())).astype(np.int32)
        per, ss, sr, rows = oracle.dispatch(ids, k, E, rc, rg)
        n = np.zeros(E, np.int64)
        for a in ids:
            n += np.bincount(a.reshape(-1), minlength=E)
        f = 0
        for e in range(E):
            sizes = sr[f:f + rc[e]]
            assert sizes.sum() == n[e] and sizes.max() - sizes.min() <= 1
            assert list(sizes) == sorted(sizes, reverse=True)
            f += rc[e]
        for g in range(G):
            got = np.concatenate([per[s][1][per[s][0] == g] for s in range(G)])
            assert np.array_equal(np.sort(got), np.arange(rows[g]))


def test_ffn_golden_and_numpy():
    g = load("ffn_small.npz")
    y = oracle.expert_ffn(g["x"], g["w1"], g["w3"], g["w2"], round_h=False, round_y=False)
    np.testing.assert_allclose(y, g["y"], rtol=1e-5, atol=1e-6)
    f = lambda a: oracle.bf16_to_f32(a).astype(np.float64)
    a, b = f(g["x"]) @ f(g["w1"]).T, f(g["x"]) @ f(g["w3"]).T
    h = a / (1 + np.exp(-a)) * b
    np.testing.assert_allclose(y, h @ f(g["w2"]).T, rtol=1e-4, atol=1e-5)


def test_layer_golden():
    g = load("gate_small.npz")
    lg = load("layer_small.npz")
    experts = [oracle.synth_expert(oracle.orc().orc_stream_key(1, 0, e, 0x65787074), 256, 256) for e in range(8)]
    y, ids, w, counts = oracle.layer_forward(g["x"], g["wg"], experts, lg["rc"], 2)
    assert np.array_equal(ids, lg["ids"]) and np.array_equal(counts, lg["counts"])
    np.testing.assert_allclose(y, lg["y"], rtol=1e-5, atol=1e-6)
    # combine == explicit weighted sum of per-expert FFNs (replica split invisible)
    ref = np.zeros_like(y)
    for t in range(y.shape[0]):
        for j in range(2):
            e = ids[t, j]
            ref[t] += w[t, j] * oracle.expert_ffn(g["x"][t:t + 1], *experts[e])[0]
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6)
def test_predict_mlp_oracle_against_numpy():
    """orc_predict_mlp vs numpy on grid weights (every product and partial sum
    exact in fp32, so summation order cannot matter)."""
    from paper_2603_06350_b200 import workload as wl
    E, k, d, T = 16, 2, 256, 200
    rng = np.random.default_rng(3)
    x = wl.tokens(T, d, E, 1, 2)
    w1 = wl.gate_weights(E, d, 1.2, 1, 1, 0)
    w2 = (rng.integers(-8, 9, (E, E)) / 8.0).astype(np.float32)
    h = np.maximum(oracle.bf16_to_f32(x).astype(np.float64) @ oracle.bf16_to_f32(w1).T.astype(np.float64), 0.0)
    out = h @ w2.T.astype(np.float64)
    want = np.zeros(E, np.int32)
    for t in range(T):
        o = out[t].copy()
        for _ in range(k):
            b = int(np.argmax(o))  # first maximum = lowest index on ties
            want[b] += 1
            o[b] = -np.inf
    assert np.array_equal(oracle.predict_mlp(x, w1, w2, k), want)
    # W2 = identity with all-positive hidden units reduces to the linear predictor
    assert oracle.predict_mlp(x, w1, np.eye(E, dtype=np.float32), k).sum() == T * k
