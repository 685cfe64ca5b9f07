"""Host planner (product C++, via the C-ABI) vs the reference (CPU only).

The product re-implements scale_experts / place_experts / ReplicaRegistry /
layer_forward_time / predict / route_tokens / percentile from scratch; plans
must be BIT-identical to the reference's on identical inputs (SURVEY §8a
"bit-exactness traps").  Checked three ways: the reference's own hand-derived
goldens (test_scaler.cpp, test_placer.cpp, test_cost_model.cpp,
test_predictor.cpp, test_config_report.cpp restated), the committed
tests/golden/planner.json produced by the compiled reference, and live
randomized comparison against oracle/_ref when it is built.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import MoeError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------ reference goldens
def test_scaler_golden_skewed_four():  # test_scaler.cpp:32-51
    p = pk.scale_experts([8, 4, 2, 2], 1.0, 8.0, 0.2)
    assert p.replica_counts == [3, 2, 1, 1]
    assert p.alloc_mem_mb == 3.0 and p.total_replicas() == 7
    assert p.split_trace == [0, 0, 1]
    assert abs(p.cv_trace[-1] - 1.0 / (4.0 * math.sqrt(3.0))) < 1e-12


def test_scaler_golden_budget_stop():  # test_scaler.cpp:53-63
    assert pk.scale_experts([10, 1, 1, 1], 1.0, 1.0, 0.1).replica_counts == [2, 1, 1, 1]


def test_scaler_balanced_zero_and_ties():  # test_scaler.cpp:65-112
    assert pk.scale_experts([5, 5, 5, 5], 1.0, 100.0).replica_counts == [1, 1, 1, 1]
    assert pk.scale_experts([0, 0, 0], 1.0, 100.0).replica_counts == [1, 1, 1]
    assert pk.scale_experts([9, 9, 0], 1.0, 100.0, 0.2).total_replicas() > 3
    assert pk.scale_experts([9, 9, 0], 1.0, 100.0, 0.2, True).replica_counts == [1, 1, 1]
    p = pk.scale_experts([6, 6, 0], 1.0, 1.0, 0.2)
    assert p.replica_counts == [2, 1, 1] and p.split_trace == [0]
    assert pk.scale_experts([6, 6], 1.0, 8.0, 0.0).replica_counts == [1, 1]


def test_scaler_validation():  # test_scaler.cpp:124-135
    with pytest.raises(ValueError):
        pk.scale_experts([], 1.0, 1.0)
    with pytest.raises(ValueError):
        pk.scale_experts([1, -2], 1.0, 1.0)
    with pytest.raises(ValueError):
        pk.scale_experts([1, 2], 1.0, 1.0, -0.5)


def _plan(loads, counts, mem=1.0):
    return pk.ScalingPlan(0, list(counts), list(loads), 0.0, mem)


def test_placer_jsq_golden():  # test_placer.cpp:48-62
    r = pk.place_experts(_plan([5, 5, 3, 2], [1, 1, 1, 1]), 2, 1e9, pk.ReplicaRegistry(0), 0)
    assert r.gpu_for == [[0], [1], [0], [1]] and r.cold_count == 4 and r.warm_count == 0


def test_placer_warm_keepalive():  # test_placer.cpp:64-84
    for it, warm, g0 in [(15, 2, 1), (16, 0, 0)]:
        reg = pk.ReplicaRegistry(5)
        pk.update_registry(reg, [1, 1], [1, 1], 2, 0, 10)
        r = pk.place_experts(_plan([10, 1], [1, 1]), 2, 1e9, reg, it)
        assert r.warm_count == warm and r.gpu_for[0][0] == g0


def test_placer_memory_and_error_message():  # test_placer.cpp:86-111
    reg = pk.ReplicaRegistry(50)
    pk.update_registry(reg, [1, 1], [0, 0], 2, 0, 0)
    with pytest.raises(MoeError, match="no GPU has memory for replica"):
        pk.place_experts(_plan([5, 4, 3], [1, 1, 1], 60.0), 2, 100.0, reg, 1)
    r = pk.place_experts(_plan([5, 4], [1, 1], 60.0), 2, 100.0, reg, 1)
    assert r.gpu_for == [[0], [1]] and r.warm_count == 1 and r.cold_count == 1
    with pytest.raises(MoeError, match="aggregate cluster capacity"):
        pk.place_experts(_plan([1, 1, 1], [1, 1, 1], 100.0), 1, 150.0, pk.ReplicaRegistry(0), 0)


def test_registry_retire():  # test_placer.cpp:113-130
    reg = pk.ReplicaRegistry(2)
    r = pk.place_experts(_plan([8, 2], [2, 1]), 2, 1e9, reg, 0)
    pk.update_registry(reg, [2, 1], r.flat(), 2, 0, 0)
    assert reg.size() == 3
    r2 = pk.place_experts(_plan([8, 2], [1, 1]), 2, 1e9, reg, 1)
    pk.update_registry(reg, [1, 1], r2.flat(), 2, 0, 1)
    assert reg.size() == 2


def test_cost_model_goldens():  # test_cost_model.cpp:66-138
    c = pk.layer_forward_time([100], [1], [0], [100], 1, 0.01, 0.001, 0.5, 0.0, 330.0)
    assert np.allclose(c[:3], [1.0, 0.1, 1.7]) and c[3] == 1 and np.isclose(c[5], 1.2 * 330.0)
    c = pk.layer_forward_time([8], [2], [0, 1], [9], 2, 1.0, 0.0, 0.0, 0.0, 1.0)
    assert np.isclose(c[0], 4.5) and np.isclose(c[2], 4.5)
    c = pk.layer_forward_time([6, 4, 2], [1, 1, 1], [0, 1, 0], [6, 4, 2], 2, 0.01, 0.002, 0.0, 0.0, 1.0)
    assert np.isclose(c[0], 0.06) and np.isclose(c[1], 0.016) and np.isclose(c[2], 0.092)
    with pytest.raises(ValueError):
        pk.layer_forward_time([5, 3], [1, 1], [0, 5], [5, 3], 2, 1, 1, 0, 0, 1)


def test_predictor_goldens():  # test_predictor.cpp:34-140
    assert pk.measure_accuracy([5, 5], [8, 2]) == pytest.approx(0.7)
    assert pk.measure_accuracy([4, 1], [8, 2]) == pytest.approx(1.0)
    assert pk.measure_accuracy([0, 0], [0, 0]) == 1.0 and pk.measure_accuracy([3, 3], [0, 0]) == 0.0
    assert pk.predict(0, [7, 0, 3])[0] == [7, 0, 3]
    pred, _ = pk.predict(1, [8000, 2000], accuracy=[0.7], iteration=0, seed=11)
    assert sum(pred) == 10000 and abs(pred[0] - 7100) < 250
    pred, fb = pk.predict(2, [7, 3], history=[[4, 4], [6, 2]], window=8)
    assert pred == [6, 4] and not fb
    pred, fb = pk.predict(2, [5, 5, 4])
    assert pred == [5, 5, 4] and fb
    pred, _ = pk.predict(1, [0, 10000], accuracy=[0.0], seed=5, popularity=[1.0, 0.0])
    assert pred[0] == 10000


def test_percentile_nearest_rank():  # test_config_report.cpp:149-159
    v = [10, 1, 9, 2, 8, 3, 7, 4, 6, 5]
    assert pk.percentile(v, 0.5) == 5.0 and pk.percentile(v, 0.95) == 10.0
    assert pk.percentile(v, 0.0) == 1.0 and pk.percentile(v, 1.0) == 10.0
    assert pk.percentile([42.0], 0.5) == 42.0
    with pytest.raises(ValueError):
        pk.percentile([], 0.5)


# ------------------------------------------------- committed reference goldens
@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "planner.json"))))
def test_planner_matches_reference_golden(case):
    p = pk.scale_experts(case["loads"], 1.0, case["cap"], case["cv"], bool(case["excl"]))
    assert p.replica_counts == case["counts"]
    assert p.alloc_mem_mb == case["alloc"]
    assert p.split_trace == case["split"]
    assert p.cv_trace == case["cv_trace"]  # bit-identical doubles
    r = pk.place_experts(p, case["G"], 1e9, pk.ReplicaRegistry(3), 0)
    assert r.flat() == case["gpu"] and r.warm_count == case["warm"] and r.cold_count == case["cold"]
    f = pk.layer_forward_time(case["loads"], case["counts"], case["gpu"], case["actual"], case["G"],
                              0.01, 0.002, 0.5, 0.0, 330.0)
    assert list(f) == case["forward"]


def test_route_tokens_matches_reference_golden():
    for entry in json.load(open(os.path.join(GOLD, "route_loads.json"))):
        T, layer, it, E, k, s, seed, drift = entry["case"]
        assert pk.route_tokens(T, layer, it, E, 8, s, seed, k, drift) == entry["loads"]


# ------------------------------------------------------------- live reference
@pytest.fixture(scope="module")
def ref():
    r = oracle.ref()
    if r is None:
        pytest.skip("reference library not built")
    return r


def test_scaler_live_random(ref):
    rng = np.random.default_rng(77)
    for _ in range(2000):
        E = int(rng.integers(1, 13))
        loads = np.where(rng.random(E) < 0.25, 0, rng.integers(0, 1000, E)).astype(np.int64)
        cap, cv, excl = float(rng.integers(0, 17)), float(rng.integers(0, 11)) / 10, int(rng.integers(0, 2))
        counts = np.zeros(E, np.int32)
        alloc, steps, ok = np.zeros(1), np.zeros(1, np.int32), np.zeros(1, np.int32)
        split, cvt = np.zeros(64, np.int32), np.zeros(64)
        assert ref.ref_scale_experts(oracle.P(loads), E, 0, 1.0, cap, cv, excl, oracle.P(counts), oracle.P(alloc),
                                     oracle.P(steps), oracle.P(split), 64, oracle.P(cvt), oracle.P(ok)) == 0
        p = pk.scale_experts(loads, 1.0, cap, cv, bool(excl))
        assert p.replica_counts == counts.tolist() and p.alloc_mem_mb == alloc[0]
        assert p.split_trace == split[:steps[0]].tolist() and p.cv_trace == cvt[:steps[0]].tolist()
        assert ok[0] == 1


def test_placer_live_sequences(ref):
    """Registry state evolves over iterations identically (warm starts,
    retirement, memory-blocked warm starts, compute-weighted queues)."""
    rng = np.random.default_rng(5)
    for trial in range(60):
        E, G = int(rng.integers(2, 12)), int(rng.integers(1, 6))
        keep = int(rng.integers(0, 4))
        cap_gpu = float(rng.choice([1e9, 4.0, 6.0]))
        incl = int(rng.integers(0, 2))
        rreg, preg = ref.ref_registry_new(keep), pk.ReplicaRegistry(keep)
        for it in range(12):
            loads = rng.integers(0, 500, E).astype(np.int64)
            counts = rng.integers(1, 3, E).astype(np.int32)
            if counts.sum() * 1.0 > G * cap_gpu:
                counts[:] = 1
            if counts.sum() > G * cap_gpu:
                continue
            gr = np.zeros(int(counts.sum()), np.int32)
            w, c = np.zeros(1, np.int32), np.zeros(1, np.int32)
            rc = ref.ref_place_experts(rreg, oracle.P(loads), oracle.P(counts), E, 0, 1.0, G, cap_gpu, it, incl,
                                       0.3, 1.0, oracle.P(gr), oracle.P(w), oracle.P(c))
            plan = _plan(loads, counts)
            if rc != 0:
                with pytest.raises((MoeError, ValueError)):
                    pk.place_experts(plan, G, cap_gpu, preg, it, bool(incl), 0.3, 1.0)
                continue
            r = pk.place_experts(plan, G, cap_gpu, preg, it, bool(incl), 0.3, 1.0)
            assert r.flat() == gr.tolist() and (r.warm_count, r.cold_count) == (w[0], c[0])
            ref.ref_update_registry(rreg, oracle.P(counts), oracle.P(gr), E, G, 0, it)
            pk.update_registry(preg, counts, gr, G, 0, it)
            assert preg.size() == ref.ref_registry_size(rreg)
        ref.ref_registry_free(rreg)


def test_predict_live(ref):
    rng = np.random.default_rng(9)
    for _ in range(200):
        E = int(rng.integers(1, 10))
        actual = rng.integers(0, 300, E).astype(np.int64)
        kind = int(rng.integers(0, 3))
        hist = rng.integers(0, 300, (int(rng.integers(0, 6)), E)).astype(np.int64)
        acc = rng.random(3)
        pop = rng.random(E) if rng.random() < 0.5 else None
        it, seed, window, dist = int(rng.integers(0, 100)), int(rng.integers(0, 1 << 40)), int(rng.integers(1, 5)), int(rng.integers(0, 4))
        out, fb = np.zeros(E, np.int64), np.zeros(1, np.int32)
        ref.ref_predict(kind, oracle.P(actual), E, 1, oracle.P(hist) if len(hist) else None, len(hist),
                        oracle.P(acc), 3, dist, 0.04, window, it, seed, oracle.P(pop) if pop is not None else None,
                        oracle.P(out), oracle.P(fb))
        got, gfb = pk.predict(kind, actual, 1, hist, acc, dist, 0.04, window, it, seed, pop)
        assert got == out.tolist() and gfb == bool(fb[0])
        assert pk.measure_accuracy(got, actual) == ref.ref_measure_accuracy(oracle.P(out), oracle.P(actual), E)


def test_route_and_percentile_live(ref):
    rng = np.random.default_rng(1)
    for _ in range(30):
        E = int(rng.integers(1, 65))
        k = int(rng.integers(1, min(8, E) + 1))
        T, it, layer = int(rng.integers(0, 2000)), int(rng.integers(0, 99)), int(rng.integers(0, 4))
        loads = np.zeros(E, np.int64)
        ref.ref_route_tokens(T, layer, it, E, 4, 1.2, 3, k, 0, oracle.P(loads))
        assert pk.route_tokens(T, layer, it, E, 4, 1.2, 3, k) == loads.tolist()
        v = rng.random(int(rng.integers(1, 300)))
        q = float(rng.random())
        assert pk.percentile(v, q) == ref.ref_percentile(oracle.P(v), len(v), q)


# ------------------------------------ baselines / cost-model rows (a8, a10, a11)
def _ref_or_skip():
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference library not built")
    return ref


def _random_plan(rng, E, G):
    loads = rng.integers(0, 5000, E).astype(np.int64)
    rc = rng.integers(1, 4, E).astype(np.int32)
    gpu = rng.integers(0, G, int(rc.sum())).astype(np.int32)
    return loads, rc, gpu


def test_static_plan_matches_reference():  # baselines.cpp:32-60
    ref = _ref_or_skip()
    rng = np.random.default_rng(11)
    for _ in range(200):
        E, G = int(rng.integers(1, 70)), int(rng.integers(1, 9))
        loads = rng.integers(0, 10000, E).astype(np.int64)
        want = np.zeros(E, np.int32)
        assert ref.ref_static_plan(oracle.P(loads), E, G, 22.0, 180000.0, oracle.P(want)) == 0
        assert pk.static_plan(loads, G, 22.0) == want.tolist()
    # a placement that does not fit: the reference's wording
    with pytest.raises(MoeError, match="static placement does not fit GPU 0"):
        pk.static_plan([1, 2, 3], 1, 100.0, 250.0)


def test_round_robin_placement_semantics():  # simulator.cpp:32-50 (anonymous there: restated)
    assert pk.round_robin_placement([2, 1, 3], 2, 10.0) == [0, 1, 0, 1, 0, 1]
    assert pk.round_robin_placement([1] * 5, 3, 10.0) == [0, 1, 2, 0, 1]
    # one replica per expert: identical to the reference's static_plan
    ref = _ref_or_skip()
    rng = np.random.default_rng(12)
    for _ in range(50):
        E, G = int(rng.integers(1, 70)), int(rng.integers(1, 9))
        want = np.zeros(E, np.int32)
        assert ref.ref_static_plan(oracle.P(np.zeros(E, np.int64)), E, G, 1.0, 1e9, oracle.P(want)) == 0
        assert pk.round_robin_placement([1] * E, G, 1.0) == want.tolist()
    with pytest.raises(MoeError, match="round-robin placement does not fit GPU 0"):
        pk.round_robin_placement([3, 1], 2, 100.0, 150.0)


def test_gpu_comm_times_matches_reference():  # cost_model.cpp:67-89
    ref = _ref_or_skip()
    rng = np.random.default_rng(13)
    for _ in range(300):
        E, G = int(rng.integers(1, 40)), int(rng.integers(1, 9))
        loads, rc, gpu = _random_plan(rng, E, G)
        beta = float(rng.choice([0.0, 0.002, 0.005, 1.0]))
        want = np.zeros(G)
        assert ref.ref_gpu_comm_times(oracle.P(loads), oracle.P(rc), oracle.P(gpu), E, G, beta, oracle.P(want)) == 0
        assert pk.gpu_comm_times(loads, rc, gpu, G, beta) == want.tolist()  # bit-identical doubles


def test_oracle_balance_time_matches_reference():  # baselines.cpp:141-154
    ref = _ref_or_skip()
    rng = np.random.default_rng(14)
    for _ in range(300):
        E, G = int(rng.integers(1, 70)), int(rng.integers(1, 9))
        actual = rng.integers(0, 20000, E).astype(np.int64)
        args = (G, float(rng.random()), float(rng.random() * 0.01), float(rng.random()), float(rng.random() * 100),
                float(rng.choice([22.0, 352.0])))
        want = np.zeros(6)
        assert ref.ref_oracle_balance_time(oracle.P(actual), E, *args, oracle.P(want)) == 0
        assert list(pk.oracle_balance_time(actual, *args)) == want.tolist()


def _ref_verify(ref, loads, rc, shares, alloc, mem, cap, cv, excl):
    sh = np.asarray(shares, np.int64).reshape(-1, 4)
    se, so = np.ascontiguousarray(sh[:, 0], np.int32), np.ascontiguousarray(sh[:, 1], np.int32)
    sn, sd = np.ascontiguousarray(sh[:, 2]), np.ascontiguousarray(sh[:, 3])
    la, rca = np.ascontiguousarray(loads, np.int64), np.ascontiguousarray(rc, np.int32)
    ok = np.zeros(1, np.int32)
    buf = oracle.C.create_string_buffer(1 << 16)
    assert ref.ref_verify_plan(oracle.P(la), len(la), oracle.P(rca), len(rca), oracle.P(se), oracle.P(so),
                               oracle.P(sn), oracle.P(sd), len(sh), alloc, mem, cap, cv, int(excl), oracle.P(ok),
                               buf, len(buf)) == 0
    return bool(ok[0]), [m for m in buf.value.decode().split("\n") if m]


def test_verify_plan_matches_reference():  # scaler.cpp:99-173, incl. broken plans
    ref = _ref_or_skip()
    rng = np.random.default_rng(15)
    n_bad = 0
    for i in range(400):
        E = int(rng.integers(1, 20))
        loads = rng.integers(0, 3000, E).astype(np.int64)
        mem, cap = 1.0, float(rng.integers(0, 2 * E))
        plan = pk.scale_experts(loads, mem, cap, 0.2)
        rc = list(plan.replica_counts)
        shares = [[e, r, int(loads[e]), rc[e]] for e in range(E) for r in range(rc[e])]
        alloc = float(plan.alloc_mem_mb)
        mut = i % 8
        if mut == 1:
            rc[int(rng.integers(E))] += 1                      # share count mismatch
        elif mut == 2 and shares:
            shares[int(rng.integers(len(shares)))][1] = 99     # out-of-range ordinal
        elif mut == 3 and shares:
            shares[int(rng.integers(len(shares)))][2] += 1     # unequal / non-conserving shares
        elif mut == 4:
            alloc += 1.0                                       # alloc mismatch
        elif mut == 5:
            rc[int(rng.integers(E))] = 0                       # replica count < 1
        elif mut == 6 and shares:
            shares[0][0] = E + 3                               # unknown expert
        elif mut == 7:
            rc = rc[:-1]                                       # wrong length
        got = pk.verify_plan(loads, rc, shares, alloc, mem, cap)
        want = _ref_verify(ref, loads, rc, shares, alloc, mem, cap, 0.2, False)
        assert got == want, (i, got, want)
        n_bad += not want[0]
    assert n_bad > 100  # the mutations exercised the failure paths


def test_apply_finetuning_matches_reference():  # predictor.cpp:188-199
    ref = _ref_or_skip()
    rng = np.random.default_rng(16)
    for _ in range(100):
        n = int(rng.integers(0, 40))
        acc = rng.random(n)
        h = float(rng.random())
        want_acc, want_ft = acc.copy(), np.zeros(max(n, 1), np.int32)
        assert ref.ref_apply_finetuning(oracle.P(want_acc), n, h, oracle.P(want_ft)) == 0
        got_acc, got_ft = pk.apply_finetuning(acc, h)
        assert got_acc == want_acc.tolist() and got_ft == [bool(v) for v in want_ft[:n]]


def test_cv_and_serverful_cost_match_reference():  # cost_model.cpp:124-139
    ref = _ref_or_skip()
    rng = np.random.default_rng(17)
    for _ in range(200):
        v = np.ascontiguousarray(rng.random(int(rng.integers(1, 50))) * rng.choice([0.0, 1.0, 1e3]))
        assert pk.coefficient_of_variation(v) == ref.ref_coefficient_of_variation(oracle.P(v), len(v))
        args = (float(rng.random() * 1e4), int(rng.integers(1, 33)), int(rng.integers(1, 65)),
                float(rng.random() * 400), float(rng.random() * 100))
        assert pk.serverful_cost(*args) == ref.ref_serverful_cost(*args)
    with pytest.raises(ValueError, match="CV of an empty sample"):
        pk.coefficient_of_variation([])
