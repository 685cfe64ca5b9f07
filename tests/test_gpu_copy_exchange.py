"""The NCCL exchange code path, run for real with G ranks on ONE B200.

MOE_EXCHANGE_COPY contexts go through exactly the forward the NCCL mode runs
(capi.cpp enqueue_forward, non-peer-memory branch): gate -> counts all-gather
(Transport::all_gather) -> host exchange plan -> dispatch into the local
receive buffer AND the send buffer -> stage_exchange's chunk loop (one
message per (peer, replica) chunk, Transport::exchange) -> grouped GEMMs ->
the reverse chunk loop into the return buffer -> combine.  Only the
transport differs from MOE_EXCHANGE_NCCL: copy-engine pulls after a host
rendezvous instead of ncclSend/ncclRecv (NCCL refuses two ranks on one GPU).
Ranks are host threads (one context each).  Every rank's output must be
BIT-IDENTICAL to a single-GPU forward on its own tokens (a row's expert output
does not depend on where it is computed), ids and counts equal the oracle's.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_EXCHANGE_COPY, MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


def _ranks(G, E, k, d, ff, Tmax, cap_replicas=0):
    group = os.urandom(128)
    mem = 3.0 * d * ff * 2 / 1e6
    return [MoELayer(1, E, k, d, ff, max_tokens=Tmax, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_COPY,
                     nccl_unique_id=group, expert_mem_mb=mem, layer_mem_cap_mb=(E + cap_replicas) * mem)
            for r in range(G)]


def _parallel(n, fn):
    with ThreadPoolExecutor(n) as ex:
        return list(ex.map(fn, range(n)))


@pytest.mark.parametrize("G,E,k,d,ff,tokens,rc,rg", [
    (2, 8, 2, 1024, 1408, [300, 170], [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 0, 1, 0, 1, 1, 0, 1]),
    (4, 8, 2, 1024, 1408, [64, 200, 1, 129], [1, 2, 1, 1, 1, 2, 1, 1], [0, 1, 2, 3, 0, 1, 2, 3, 0, 1]),
    (4, 16, 2, 1024, 1408, [128, 0, 64, 200], [1] * 16, [e % 4 for e in range(16)]),
    (8, 64, 8, 2048, 1408, [32] * 8, [1] * 60 + [2, 3, 1, 2], [i % 8 for i in range(68)]),
])
def test_copy_transport_fixed_placement(cuda, G, E, k, d, ff, tokens, rc, rg):
    import torch
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    Tmax = max(max(tokens), 1)
    ms = _ranks(G, E, k, d, ff, Tmax)
    one = MoELayer(1, E, k, d, ff, max_tokens=Tmax)
    for m in ms + [one]:
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
    for m in ms:
        m.set_placement(0, rc, rg)
    xs = [wl.tokens(tokens[r], d, E, 1, 70 + r) for r in range(G)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    yd = [torch.zeros((max(t, 1), d), dtype=torch.int16, device=cuda)[:t] for t in tokens]
    for it in range(3):  # repeated forwards: buffer reuse across steps
        sts = _parallel(G, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it, stats=True))
        torch.cuda.synchronize()
        assert sum(st.rows_local for st in sts) == k * sum(tokens)
        assert sum(st.rows_sent for st in sts) > 0  # rows really crossed ranks
        for r in range(G):
            T = tokens[r]
            if T == 0:
                continue
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
            ids = ms[r].read_buffer(4, np.int32, (T, k))
            y_ref, ids_o, _, counts_o = oracle.layer_forward(xs[r], wg, experts, [1] * E, k)
            assert np.array_equal(ids, ids_o)
            assert np.array_equal(np.array(sts[r].counts[:E]), counts_o)
            y = oracle.bf16_to_f32(yd[r].cpu().numpy().view(np.uint16))
            assert row_rel_err(y, y_ref) <= 2e-2
    for m in ms + [one]:
        m.close()


def test_copy_transport_sync_planner(cuda):
    """MOE_PLAN_SYNC at G=4 through the NCCL-path forward: all-gathered
    histograms, identical host plans on every rank, straggler replicas."""
    import torch
    G, E, k, d, ff, T = 4, 16, 2, 1024, 1408, 192
    ms = _ranks(G, E, k, d, ff, T, cap_replicas=6)
    one = MoELayer(1, E, k, d, ff, max_tokens=T)
    for m in ms + [one]:
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 90 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    extra = []
    for it in range(4):
        wg = wl.gate_weights(E, d, 1.6, 1, 0, it)
        for m in ms + [one]:
            m.set_gate(0, wg)
        sts = _parallel(G, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_SYNC, it, stats=True))
        torch.cuda.synchronize()
        plans = [m.placement(0) for m in ms]
        assert all(np.array_equal(p[0], plans[0][0]) and np.array_equal(p[1], plans[0][1]) for p in plans)
        extra.append(sts[0].replica_count - E)
        assert sum(st.rows_local for st in sts) == k * G * T
        for r in range(G):
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    assert max(extra) > 0  # the planner added replicas
    for m in ms + [one]:
        m.close()
