"""Peer-memory expert parallelism (MOE_EXCHANGE_P2P) with G ranks sharing ONE
B200 (the pool has one GPU per call).

Each rank is a full context: its dispatch kernel stores rows straight into the
owning rank's received-rows buffer, its combine reads expert outputs from the
owner, and device flags order the phases — the same code that runs over
NVLink between GPUs.  Ranks are driven by host threads (one process, plain
pointers) and by separate processes (CUDA IPC handles).

A row's expert output does not depend on which rank computes it (the GEMM's
per-row K loop is the same wherever the row lands), so every rank's output
must be BIT-IDENTICAL to a single-GPU forward on its own tokens, whatever
the placement; ids and counts are checked against the oracle.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import (MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MOE_PLAN_PREDICTED, MOE_PLAN_SYNC, MoeError,
                                   MoELayer)
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ranks(G, E, k, d, ff, Tmax, cap_replicas=0, **kw):
    mem = 3.0 * d * ff * 2 / 1e6
    ms = [MoELayer(1, E, k, d, ff, max_tokens=Tmax, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   expert_mem_mb=mem, layer_mem_cap_mb=(E + cap_replicas) * mem, **kw) for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
    return ms


def _single(E, k, d, ff, Tmax):
    mem = 3.0 * d * ff * 2 / 1e6
    return MoELayer(1, E, k, d, ff, max_tokens=Tmax, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)


def _parallel(ms, fn):
    with ThreadPoolExecutor(len(ms)) as ex:
        return list(ex.map(fn, range(len(ms))))


@pytest.mark.parametrize("G,E,k,d,ff,tokens,rc,rg", [
    (2, 8, 2, 1024, 1408, [256, 200], [1] * 8, [0, 1, 0, 1, 0, 1, 0, 1]),
    (2, 8, 2, 1024, 1408, [300, 1], [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 1, 0, 1, 0, 0, 1, 1]),
    (4, 16, 2, 1024, 1408, [128, 64, 0, 200], [1] * 16, [e % 4 for e in range(16)]),
    (4, 64, 8, 2048, 1408, [64, 64, 64, 64], [1] * 62 + [3, 2], [e % 4 for e in range(62)] + [0, 1, 2, 3, 3]),
])
def test_p2p_fixed_placement_bit_identical(cuda, G, E, k, d, ff, tokens, rc, rg):
    import torch
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    Tmax = max(max(tokens), 1)
    ms = _ranks(G, E, k, d, ff, Tmax)
    one = _single(E, k, d, ff, Tmax)
    for m in ms + [one]:
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
    for m in ms:
        m.set_placement(0, rc, rg)
    xs = [wl.tokens(tokens[r], d, E, 1, 70 + r) for r in range(G)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    yd = [torch.zeros((max(t, 1), d), dtype=torch.int16, device=cuda)[:t] for t in tokens]
    for it in range(3):  # repeated forwards exercise the epoch flags and buffer reuse
        sts = _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it, stats=True))
        torch.cuda.synchronize()
        assert sum(st.rows_local for st in sts) == k * sum(tokens)
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


def test_p2p_sync_planner_replicas(cuda):
    """MOE_PLAN_SYNC at G=4: every rank runs scale/place on the all-gathered
    histogram (identical decisions), straggler replicas split hot experts over
    ranks, gates change every iteration; outputs stay bit-identical to G=1."""
    import torch
    G, E, k, d, ff, T = 4, 16, 2, 1024, 1408, 192
    ms = _ranks(G, E, k, d, ff, T, cap_replicas=6)
    one = _single(E, k, d, ff, T)
    for m in ms + [one]:
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 90 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    replicas = []
    for it in range(4):
        wg = wl.gate_weights(E, d, 1.6, 1, 0, it)
        for m in ms + [one]:
            m.set_gate(0, wg)
        sts = _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_SYNC, it, stats=True))
        torch.cuda.synchronize()
        assert len({st.replica_count for st in sts}) == 1  # same plan on every rank
        replicas.append(sts[0].replica_count)
        assert sum(st.rows_local for st in sts) == k * G * T
        for r in range(G):
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    assert max(replicas) > E  # the planner did add straggler replicas
    for m in ms + [one]:
        m.close()


def test_p2p_rank_out_of_step_times_out(cuda, monkeypatch):
    """A rank whose peers never arrive fails instead of hanging the GPU."""
    import torch
    monkeypatch.setenv("MOE_P2P_TIMEOUT_MS", "300")
    E, k, d, ff, T = 8, 2, 256, 256, 64
    ms = _ranks(2, E, k, d, ff, T)
    for m in ms:
        m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    x = torch.from_numpy(wl.tokens(T, d, E, 1, 0).view(np.int16)).to(cuda)
    y = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    with pytest.raises(MoeError, match="timed out"):  # device-planned: surfaces at the next sync point
        ms[0].forward(0, x, y, MOE_PLAN_FIXED, 0)
        ms[0].sync()
    ms[0].close()
    ms[1].close()


@pytest.mark.parametrize("residency", [0, 1])
def test_p2p_two_processes_ipc(cuda, tmp_path, residency):
    """Two processes on the same device, slabs shared with CUDA IPC handles
    exchanged over gloo (tests/p2p_worker.py); each checks itself against a
    single-GPU forward.  residency=1: MOE_RESIDENCY_PLACED, so cold replicas are
    copied out of the peer process's IPC-mapped weight slots."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29731 + residency), PYTHONPATH=ROOT)
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "p2p_worker.py"), str(r), "2",
                               str(residency)],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(2)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append(out.decode(errors="replace"))
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
        assert "P2P-IPC OK" in o, o[-3000:]
    if residency:  # some replica was copied across the process boundary
        copies = [int(o.split("weight copies")[-1].split()[0]) for o in outs]
        assert sum(copies) > 0, copies


def test_p2p_predicted_planning_ahead(cuda):
    """MOE_PLAN_PREDICTED at G=2 over a 3-layer stack: layer l's fused
    predictor scores layer l+1, every rank plans layer l+1 from the gathered
    predicted histogram while layer l finishes, and layer l+1 runs with the
    ON-DEVICE exchange plan (no host round trip).  Layer 0 bootstraps from
    history on the host.  Outputs stay bit-identical to G = 1."""
    import torch
    G, L, E, k, d, ff, T = 2, 3, 16, 2, 1024, 1408, 160
    mem = 3.0 * d * ff * 2 / 1e6
    ms = [MoELayer(L, E, k, d, ff, max_tokens=T, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   num_predictor_targets=1, expert_mem_mb=mem, layer_mem_cap_mb=(E + 4) * mem) for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
    one = MoELayer(L, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    gates = [wl.gate_weights(E, d, 1.5, 1, l, 0) for l in range(L)]
    for m in ms + [one]:
        for l in range(L):
            m.set_gate(l, gates[l])
            for e in range(E):
                m.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    for m in ms:
        for l in range(L - 1):
            m.set_predictor(l, 0, gates[l + 1])  # scores layer l+1's routing from layer l's input
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 500 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [[torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(L)] for _ in range(G)]
    sources = []
    for it in range(3):
        def rank_stack(r):
            out = []
            for l in range(L):
                out.append(ms[r].forward(l, xd[r], yd[r][l], MOE_PLAN_PREDICTED, it, stats=True))
            return out
        sts = _parallel(ms, rank_stack)
        torch.cuda.synchronize()
        sources.append([st.plan_source for st in sts[0]])
        for r in range(G):
            assert [st.plan_source for st in sts[r]] == sources[-1]
            for l in range(L):
                y1 = torch.zeros((T, d), dtype=torch.int16, device=cuda)
                one.forward(l, xd[r], y1, MOE_PLAN_FIXED, it)
                one.sync()
                assert torch.equal(yd[r][l], y1), (it, r, l)
        assert sum(st.rows_local for st in [sts[r][1] for r in range(G)]) == k * G * T
    assert all(src[0] == 3 and src[1] == 2 and src[2] == 2 for src in sources), sources
    for m in ms + [one]:
        m.close()


def test_p2p_graph_replay(cuda):
    """A peer-memory layer with a fixed placement replays as one CUDA graph per
    rank (epochs live in device memory); results equal the eager G = 1 layer."""
    import torch
    G, E, k, d, ff, T = 2, 8, 2, 1024, 1408, 96
    ms = _ranks(G, E, k, d, ff, T, cuda_graphs=True)
    one = _single(E, k, d, ff, T)
    for m in ms + [one]:
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    for m in ms:
        m.set_placement(0, [1, 2, 1, 1, 1, 1, 1, 1], [0, 1, 0, 1, 1, 0, 1, 0, 1])
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 600 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    for it in range(5):
        wg = wl.gate_weights(E, d, 1.3, 1, 0, it)
        for m in ms + [one]:
            m.set_gate(0, wg)
        _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it))
        for m in ms:
            m.sync()
        for r in range(G):
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    for m in ms + [one]:
        m.close()


def test_p2p_predicted_planning_distance_two(cuda):
    """As test_p2p_predicted_planning_ahead with predictor distance 2 over 4
    layers at G=2: layers 2-3 run the on-device exchange plan from placements
    decided two layers earlier; outputs bit-identical to G = 1."""
    import torch
    G, L, E, k, d, ff, T, dist = 2, 4, 16, 2, 1024, 1408, 128, 2
    mem = 3.0 * d * ff * 2 / 1e6
    ms = [MoELayer(L, E, k, d, ff, max_tokens=T, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   num_predictor_targets=1, predictor_distance=dist, expert_mem_mb=mem,
                   layer_mem_cap_mb=(E + 4) * mem) for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
    one = MoELayer(L, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    gates = [wl.gate_weights(E, d, 1.5, 1, l, 0) for l in range(L)]
    for m in ms + [one]:
        for l in range(L):
            m.set_gate(l, gates[l])
            for e in range(E):
                m.load_expert(l, e, *wl.expert_weights(d, ff, 1, l, e))
    for m in ms:
        for l in range(L - dist):
            m.set_predictor(l, 0, gates[l + dist])
    xd = [torch.from_numpy(wl.tokens(T, d, E, 1, 800 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [[torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(L)] for _ in range(G)]
    for it in range(3):
        def rank_stack(r):
            return [ms[r].forward(l, xd[r], yd[r][l], MOE_PLAN_PREDICTED, it, stats=True) for l in range(L)]
        sts = _parallel(ms, rank_stack)
        torch.cuda.synchronize()
        for r in range(G):
            assert [st.plan_source for st in sts[r]] == [3, 3, 2, 2]
            for l in range(L):
                y1 = torch.zeros((T, d), dtype=torch.int16, device=cuda)
                one.forward(l, xd[r], y1, MOE_PLAN_FIXED, it)
                one.sync()
                assert torch.equal(yd[r][l], y1), (it, r, l)
    for m in ms + [one]:
        m.close()


@pytest.mark.parametrize("variant", ["2sm", "1sm"])
def test_p2p_prefill_kernels_bit_identical(cuda, monkeypatch, variant):
    """The prefill K4 kernels (the 2-SM default and the 1-SM one) behind the
    peer-memory exchange: G=2 ranks with straggler replicas split across them,
    every rank's output bit-identical to one GPU running the same kernel."""
    import torch
    monkeypatch.setenv("MOE_GEMM_VARIANT", variant)
    G, E, k, d, ff, T = 2, 8, 2, 1024, 1408, 1500
    rc, rg = [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 1, 0, 1, 0, 0, 1, 1]
    ms = _ranks(G, E, k, d, ff, T)
    one = _single(E, k, d, ff, T)
    wg = wl.gate_weights(E, d, 1.3, 1, 0, 0)
    for m in ms + [one]:
        m.set_gate(0, wg)
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    for m in ms:
        m.set_placement(0, rc, rg)
    xs = [wl.tokens(T, d, E, 1, 300 + r) for r in range(G)]
    xd = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs]
    yd = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(G)]
    for it in range(2):
        sts = _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it, stats=True))
        torch.cuda.synchronize()
        assert sum(st.rows_local for st in sts) == k * G * T and sts[0].rows_sent > 0
        for r in range(G):
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (variant, it, r)
    y = oracle.bf16_to_f32(yd[0].cpu().numpy().view(np.uint16))
    y_ref = oracle.layer_forward(xs[0], wg, [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)], [1] * E, k)[0]
    assert row_rel_err(y, y_ref) <= 2e-2
    for m in ms + [one]:
        m.close()


def test_p2p_forwards_replayed_as_cuda_graphs(cuda):
    """Two ranks on the peer-memory exchange, FIXED placement (device-planned):
    each rank records its forward as a CUDA graph (moe_graph_begin / end) and the
    replays — re-routed between them by device-side gate updates — stay
    bit-identical to single-GPU eager forwards on the same tokens (the epoch
    lives in device memory, so every replay opens a fresh exchange epoch)."""
    import torch
    G, E, k, d, ff = 2, 8, 2, 1024, 1408
    tokens = [256, 200]
    rc, rg = [1] * E, [e % G for e in range(E)]
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    gates = [wl.gate_weights(E, d, 1.2, 1, 0, it) for it in range(3)]
    gd = [torch.from_numpy(g.view(np.int16)).to(cuda) for g in gates]
    ms = _ranks(G, E, k, d, ff, max(tokens))
    one = _single(E, k, d, ff, max(tokens))
    for m in ms + [one]:
        m.set_gate(0, gates[0])
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
    for m in ms:
        m.set_placement(0, rc, rg)
    xd = [torch.from_numpy(wl.tokens(tokens[r], d, E, 1, 90 + r).view(np.int16)).to(cuda) for r in range(G)]
    yd = [torch.zeros((t, d), dtype=torch.int16, device=cuda) for t in tokens]
    _parallel(ms, lambda r: ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, 0))  # warm: placement tables in place
    torch.cuda.synchronize()
    gids = []
    for r in range(G):
        ms[r].graph_begin()
        ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, 0)
        gids.append(ms[r].graph_end())
    for it in (1, 2, 0, 1):
        for m in ms + [one]:
            m.set_gate_device(0, gd[it])
        _parallel(ms, lambda r: ms[r].graph_launch(gids[r]))
        torch.cuda.synchronize()
        for r in range(G):
            y1 = torch.zeros_like(yd[r])
            one.forward(0, xd[r], y1, MOE_PLAN_FIXED, it)
            one.sync()
            assert torch.equal(yd[r], y1), (it, r)
    for m in ms + [one]:
        m.close()
