"""The reference's acceptance properties for the planner (proj/tests/acceptance.cpp
checks 1 and 2), run on the shipped host planner (libmoe_b200's moeless::
restatement, bit-identical to the reference per test_planner_parity.py).

Check 1 (acceptance.cpp:141-193): hand-derived scaler plans, then 10 000 random
instances: termination bound, max-share monotonicity, budget safety,
conservation of replicas, determinism.
Check 2 (acceptance.cpp:196-241): cold JSQ placement of scaled plans stays
within the greedy makespan bound (4/3 - 1/(3G)) * max(total/G, max share) on
1000 instances.  Instances are drawn with numpy here (the reference draws them
from its keyed mt19937_64); the properties hold for every instance.
"""
import math

import numpy as np

from paper_2603_06350_b200 import ReplicaRegistry, place_experts, scale_experts


def test_scaler_hand_goldens():  # acceptance.cpp:145-160
    plan = scale_experts([8, 4, 2, 2], expert_mem_mb=1.0, layer_mem_cap_mb=8.0, cv_threshold=0.2)
    assert plan.replica_counts == [3, 2, 1, 1]
    assert abs(plan.cv_trace[-1] - 1.0 / (4.0 * math.sqrt(3.0))) < 1e-12
    plan = scale_experts([10, 1, 1, 1], expert_mem_mb=1.0, layer_mem_cap_mb=1.0, cv_threshold=0.2)
    assert plan.replica_counts == [2, 1, 1, 1]


def test_scaler_properties_10000_instances():  # acceptance.cpp:162-190
    rng = np.random.default_rng(77)
    for _ in range(10000):
        E = int(rng.integers(1, 13))
        loads = [0 if rng.integers(4) == 0 else int(rng.integers(1000)) for _ in range(E)]
        cap = float(rng.integers(17))
        cv = 0.1 * int(rng.integers(11))
        excl = bool(rng.integers(2))
        plan = scale_experts(loads, 1.0, cap, cv, excl)
        steps = len(plan.split_trace)
        assert plan.total_replicas() == E + steps
        assert steps <= int(cap / 1.0)
        assert plan.alloc_mem_mb <= cap + 1e-9
        assert all(r >= 1 for r in plan.replica_counts)
        # max share after each split never grows (splits always hit a max-share expert)
        counts = [1] * E
        prev = max(l / c for l, c in zip(loads, counts))
        for e in plan.split_trace:
            counts[e] += 1
            cur = max(l / c for l, c in zip(loads, counts))
            assert cur <= prev
            prev = cur
        assert counts == plan.replica_counts
        assert scale_experts(loads, 1.0, cap, cv, excl).replica_counts == plan.replica_counts


def test_cold_placement_within_greedy_bound_1000_instances():  # acceptance.cpp:196-241
    rng = np.random.default_rng(2024)
    worst = 0.0
    for i in range(1000):
        G = 2 + int(rng.integers(4))
        E = 2 * G + int(rng.integers(9))
        s = 0.8 + 0.6 * rng.random()
        w = [1 + int(1000.0 / (e + 1) ** s) for e in range(E)]
        rng.shuffle(w)
        plan = scale_experts(w, 1.0, float(rng.integers(2 * G)), 0.2)
        placed = place_experts(plan, G, 1e9, ReplicaRegistry(0), 0)
        sums = [0.0] * G
        total, max_share = 0.0, 0.0
        for e, per in enumerate(placed.gpu_for):
            share = plan.loads[e] / plan.replica_counts[e]
            for g in per:
                sums[g] += share
                total += share
                max_share = max(max_share, share)
        bound = (4.0 / 3.0 - 1.0 / (3.0 * G)) * max(total / G, max_share)
        worst = max(worst, max(sums) / bound)
        assert max(sums) <= bound * (1 + 1e-12), (i, max(sums), bound)
    assert worst <= 1.0


def test_noisy_predictor_hits_configured_accuracy():  # acceptance.cpp:379-404
    from paper_2603_06350_b200 import measure_accuracy, predict
    actual = [15000] * 8 + [0] * 8
    popularity = [0.0] * 8 + [0.125] * 8  # misplaced tokens never overlap the actual mass
    for a in (0.7, 0.8, 0.9):
        pred, _ = predict(1, actual, layer=0, accuracy=[a], distance=1, iteration=5, seed=99,
                          popularity=popularity)
        assert abs(measure_accuracy(pred, actual) - a) <= 0.02, a
