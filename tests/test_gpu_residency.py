"""Expert weight residency driven by the placement (MOE_RESIDENCY_PLACED,
SURVEY.md §8f f2) with G ranks sharing one B200 over the peer-memory path.

Each rank keeps only its home experts (e mod G) plus a few cache slots per
layer; a replica placed on a rank whose expert is not resident there is copied
from the home rank's slot (peer memory, copy engine) before the layer's GEMMs.
Outputs must stay BIT-IDENTICAL to a single-GPU layer with every expert
resident, whatever was copied or evicted; warm hits (the ReplicaRegistry
keep-alive, placer.cpp:84-92) must avoid copies.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle

from paper_2603_06350_b200 import (MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MOE_PLAN_PREDICTED, MOE_PLAN_SYNC, MoeError,
                                   MoELayer)
from paper_2603_06350_b200 import _capi
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu
PLACED = _capi.MOE_RESIDENCY_PLACED


def _ranks(G, L, E, k, d, ff, T, cap_replicas=0, **kw):
    mem = 3.0 * d * ff * 2 / 1e6
    ms = [MoELayer(L, E, k, d, ff, max_tokens=T, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   expert_mem_mb=mem, layer_mem_cap_mb=(E + cap_replicas) * mem, residency=PLACED, **kw)
          for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
    return ms


def _single(L, E, k, d, ff, T):
    mem = 3.0 * d * ff * 2 / 1e6
    return MoELayer(L, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)


def _parallel(ms, fn):
    with ThreadPoolExecutor(len(ms)) as ex:
        return list(ex.map(fn, range(len(ms))))


def _check_oracle(x, wg, experts, k, y_dev, ids_dev_layer=None):
    """Output of one rank vs the CPU oracle on its tokens: per-token relative error <= 2e-2."""
    y = oracle.bf16_to_f32(y_dev.cpu().numpy().view(np.uint16))
    y_ref, ids_o, _, counts_o = oracle.layer_forward(x, wg, experts, [1] * len(experts), k, round_h=True)
    scale = np.maximum(np.max(np.abs(y_ref), axis=1), 1e-6)
    assert float(np.max(np.max(np.abs(y - y_ref), axis=1) / scale)) <= 2e-2
    return counts_o


class RefPlanner:
    """The compiled reference's scale_experts -> place_experts -> update_registry
    sequence (placer.cpp:11-43,45-130) on the all-gathered loads."""

    def __init__(self, keep_alive=50):
        self.ref = oracle.ref()
        self.reg = self.ref.ref_registry_new(keep_alive) if self.ref else None

    def step(self, loads, E, G, mem, cap, it):
        ref = self.ref
        la = np.ascontiguousarray(loads, np.int64)
        rc = np.zeros(E, np.int32)
        assert ref.ref_scale_experts(oracle.P(la), E, 0, mem, cap, 0.2, 0, oracle.P(rc), None, None, None, 0,
                                     None, None) == 0
        gpu = np.zeros(int(rc.sum()), np.int32)
        warm, cold = np.zeros(1, np.int32), np.zeros(1, np.int32)
        assert ref.ref_place_experts(self.reg, oracle.P(la), oracle.P(rc), E, 0, mem, G, 180000.0, it, 0, 0.0, 1.0,
                                     oracle.P(gpu), oracle.P(warm), oracle.P(cold)) == 0
        assert ref.ref_update_registry(self.reg, oracle.P(rc), oracle.P(gpu), E, G, 0, it) == 0
        return rc, gpu, int(warm[0]), int(cold[0])


def _check_residency(m, layer, rc, rg, G, rank):
    slot_of, n_slots = m.residency(layer)
    E = len(rc)
    home = (E + G - 1) // G
    f = 0
    for e in range(E):
        here = any(rg[f + r] == rank for r in range(rc[e]))
        f += rc[e]
        if e % G == rank:
            assert slot_of[e] == e // G  # home experts never move
        elif here:
            assert home <= slot_of[e] < n_slots, (e, slot_of[e])
    res = slot_of[slot_of >= 0]
    assert len(set(res.tolist())) == len(res)  # one expert per slot


def test_placed_sync_planner_bit_identical(cuda):
    """G=4, MOE_PLAN_SYNC: straggler replicas land off their home rank and are
    copied in; later iterations reuse cached replicas (warm)."""
    import torch
    G, E, k, d, ff, T = 4, 16, 2, 1024, 1408, 192
    ms = _ranks(G, 1, E, k, d, ff, T, cap_replicas=6)
    one = _single(1, E, k, d, ff, T)
    for m in ms + [one]:
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    xs = [wl.tokens(T, d, E, 1, 90 + r) for r in range(G)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    mem = 3.0 * d * ff * 2 / 1e6
    refp = RefPlanner(50)
    copies, hits = 0, 0
    for it in range(6):
        wg = wl.gate_weights(E, d, 1.6, 1, 0, it // 2)  # the routing changes every other iteration
        for m in ms + [one]:
            m.set_gate(0, wg)
        sts = _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_SYNC, it, stats=True))
        torch.cuda.synchronize()
        # outputs and histograms vs the oracle; the placement and its warm/cold split
        # vs the compiled reference's planner + registry on the same global loads
        loads = sum(_check_oracle(xs[r], wg, experts, k, yd[r]).astype(np.int64) for r in range(G))
        if refp.ref is not None:
            rc, gpu, warm, cold = refp.step(loads, E, G, mem, (E + 6) * mem, it)
            prc, prg = ms[0].placement(0)
            assert np.array_equal(prc, rc) and np.array_equal(prg, gpu), it
            assert (sts[0].warm_count, sts[0].cold_count) == (warm, cold), it
            for r in range(G):  # a replica off its home rank is resident after the forward
                _check_residency(ms[r], 0, rc, gpu, G, r)
        for r in range(G):
            st = sts[r]
            copies += st.weight_copies
            hits += st.weight_hits
            if st.weight_copies:
                assert st.weight_copy_ms > 0 and st.weight_copy_mb > 0
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    assert copies > 0 and hits > 0, (copies, hits)
    for m in ms + [one]:
        m.close()


def test_placed_eviction_with_small_cache(cuda):
    """G=2, 2 cache slots: fixed placements rotate non-home experts through
    rank 0, forcing evictions (LRU); every forward stays exact."""
    import torch
    G, E, k, d, ff, T = 2, 8, 2, 1024, 1408, 128
    ms = _ranks(G, 1, E, k, d, ff, T, replica_slots=2)
    one = _single(1, E, k, d, ff, T)
    for m in ms + [one]:
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
        m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
    xs = [wl.tokens(T, d, E, 1, 700 + r) for r in range(G)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    # odd experts are home on rank 1; each placement moves two of them to rank 0
    moves = [(1, 3), (5, 7), (1, 5), (3, 7), (1, 3)]
    for it, mv in enumerate(moves):
        rc = [1] * E
        rg = [e % G for e in range(E)]
        for e in mv:
            rg[e] = 0
        for m in ms:
            m.set_placement(0, rc, rg)
        _check_residency(ms[0], 0, rc, rg, G, 0)
        sts = _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it, stats=True))
        torch.cuda.synchronize()
        # LRU over 2 slots: (1,3) cold; (5,7) evict both; (1,5) 5 warm; (3,7) evict both; (1,3) 3 warm
        assert (sts[0].weight_copies, sts[0].weight_hits) == [(2, 0), (2, 0), (1, 1), (2, 0), (1, 1)][it]
        assert sts[1].weight_copies == 0
        for r in range(G):
            _check_oracle(xs[r], wg, experts, k, yd[r])  # copied-in weights compute the oracle's layer
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    # a placement that needs more non-home experts on rank 0 than it has slots
    rg = [0] * E
    before = ms[0].residency(0)[0].copy()
    with pytest.raises(MoeError, match="no replica slot free"):
        ms[0].set_placement(0, [1] * E, rg)
    assert np.array_equal(ms[0].residency(0)[0], before)  # the previous residency stays in force
    for m in ms + [one]:
        m.close()


def test_placed_predicted_prewarm(cuda):
    """MOE_PLAN_PREDICTED over a 3-layer stack at G=2: layer l+1's placement
    (and its replica copies) is decided from layer l's predictor ahead of the
    layer; outputs stay exact."""
    import torch
    G, L, E, k, d, ff, T = 2, 3, 16, 2, 1024, 1408, 160
    ms = _ranks(G, L, E, k, d, ff, T, cap_replicas=4, num_predictor_targets=1)
    one = _single(L, E, k, d, ff, T)
    gates = [wl.gate_weights(E, d, 1.5, 1, l, 0) for l in range(L)]
    for m in ms + [one]:
        for l in range(L):
            m.set_gate(l, gates[l])
            for e in range(E):
                m.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    for m in ms:
        for l in range(L - 1):
            m.set_predictor(l, 0, gates[l + 1])
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 500 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [[torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(L)] for _ in range(G)]
    copies = 0
    for it in range(3):
        def rank_stack(r):
            return [ms[r].forward(l, xd[r], yd[r][l], MOE_PLAN_PREDICTED, it, stats=True) for l in range(L)]
        sts = _parallel(ms, rank_stack)
        torch.cuda.synchronize()
        copies += sum(st.weight_copies for row in sts for st in row)
        for r in range(G):
            for l in range(L):
                y1 = torch.zeros((T, d), dtype=torch.int16, device=cuda)
                one.forward(l, xd[r], y1, MOE_PLAN_FIXED, it)
                one.sync()
                assert torch.equal(yd[r][l], y1), (it, r, l)
    assert copies > 0
    for m in ms + [one]:
        m.close()
