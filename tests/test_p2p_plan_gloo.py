"""Peer-memory exchange plan (MOE_EXCHANGE_P2P) on CPU: world_size 2-4 over gloo.

Every rank builds the DIRECT plan with the product host code
(exchange_plan.cpp via moe_exchange_plan_direct): for each replica, the rank
that hosts it and the row base inside THAT rank's received-rows buffer.  The
test plays the dispatch kernel's remote stores (each assignment's row goes to
(target, row_base + global rank)) through gloo messages, checks that every
rank's buffer is covered exactly once and that segments hold their replica's
rows in (source rank, token) order, runs the oracle expert FFN per segment,
plays the combine's remote loads, and compares every rank's output with the
single-process oracle layer.  The direct plan must also agree with the
chunked NCCL plan on every segment's position.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

E, K, D, FF = 8, 2, 256, 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rc, rg, tokens_per_rank, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        wg = wl.gate_weights(E, D, 1.2, 1, 0, 0)
        experts = [wl.expert_weights(D, FF, 1, 0, e) for e in range(E)]
        T = tokens_per_rank[rank]
        x = wl.tokens(T, D, E, 1, 300 + rank)
        ids, w, counts = oracle.gate(x, wg, K)
        parts = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(counts.astype(np.int32)))
        counts_all = torch.stack(parts).numpy()
        plan = pk.exchange_plan_direct(world, rank, counts_all, rc, rg)
        chunked = pk.exchange_plan(world, rank, counts_all, rc, rg)
        assert plan["rows_local"] == chunked["rows_local"]
        assert plan["rep_target"] == [int(g) for g in rg]

        rep_base = np.concatenate([[0], np.cumsum(rc)])
        n = counts_all.sum(0)
        start, size = np.zeros(len(rg), np.int64), np.zeros(len(rg), np.int64)
        for e in range(E):
            q_, r_ = divmod(int(n[e]), int(rc[e]))
            for r in range(rc[e]):
                start[rep_base[e] + r] = r * q_ + min(r, r_)
                size[rep_base[e] + r] = q_ + (1 if r < r_ else 0)
        for f in range(len(rg)):  # the segment layout both plans describe
            if rg[f] == rank:
                assert plan["rep_row_base"][f] + start[f] == chunked["seg_start"][f]
        src_off = counts_all[:rank].sum(0)

        # dispatch: every assignment -> (target rank, row in the target's buffer)
        outbox = [[] for _ in range(world)]
        where = {}
        seen = {e: 0 for e in range(E)}
        for t in range(T):
            for j in range(K):
                e = int(ids[t, j])
                # stable rank of (t, e) among this rank's assignments of e
                gr = int(src_off[e]) + int(np.sum(ids[:t] == e))
                seen[e] += 1
                f = rep_base[e] + int(np.searchsorted(start[rep_base[e]:rep_base[e + 1]], gr, side="right") - 1)
                tgt, row = plan["rep_target"][f], plan["rep_row_base"][f] + gr
                outbox[tgt].append((row, x[t]))
                where[(t, j)] = (tgt, row)
        assert all(seen[e] == counts[e] for e in range(E))
        gathered = [None] * world  # the remote stores: every rank's outbox, per destination
        dist.all_gather_object(gathered, outbox)
        xp = np.zeros((plan["rows_local"], D), np.uint16)
        hits = np.zeros(plan["rows_local"], np.int32)
        for src in range(world):
            for row, data in gathered[src][rank]:
                xp[row] = data
                hits[row] += 1
        assert np.all(hits == 1), "every received row written exactly once"

        # experts on the local segments (replica order)
        y_rows = np.zeros((plan["rows_local"], D), np.float32)
        for f in range(len(rg)):
            if rg[f] == rank and size[f] > 0:
                e = int(np.searchsorted(rep_base, f, side="right") - 1)
                s0 = plan["rep_row_base"][f] + start[f]
                y_rows[s0:s0 + size[f]] = oracle.expert_ffn(xp[s0:s0 + size[f]], *experts[e])
        yb = oracle.f32_to_bf16(y_rows)

        # combine: remote loads from the owners' outputs
        all_y = [None] * world
        dist.all_gather_object(all_y, yb)
        y = np.zeros((T, D), np.float32)
        for t in range(T):
            for j in range(K):
                tgt, row = where[(t, j)]
                y[t] += w[t, j] * oracle.bf16_to_f32(all_y[tgt][row])
        y_ref, ids_ref, _, _ = oracle.layer_forward(x, wg, experts, [1] * E, K)
        assert np.array_equal(ids, ids_ref)
        err = row_rel_err(y, y_ref)
        q.put((rank, err, plan["rows_local"], plan["rows_send"]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # surface the failure to the parent
        import traceback
        q.put((rank, "ERR " + traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("world,rc,rg,tokens", [
    (2, [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 0, 1, 0, 1, 1, 0, 1], [40, 33]),
    (3, [3, 1, 2, 1, 1, 1, 1, 1], [0, 1, 2, 2, 0, 1, 1, 0, 2, 0, 1], [17, 30, 0]),
    (4, [1, 2, 1, 1, 4, 1, 1, 1], [0, 1, 3, 2, 3, 0, 1, 2, 3, 0, 1, 2], [20, 8, 31, 13]),
])
def test_direct_plan_over_gloo(world, rc, rg, tokens):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, np.array(rc, np.int32), np.array(rg, np.int32),
                                               tokens, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    total_rows = sent = 0
    for rank, err, rows_local, rows_send in res:
        assert not isinstance(err, str), err
        assert err <= 2e-2
        total_rows += rows_local
        sent += rows_send
    assert total_rows == K * sum(tokens)
    assert 0 < sent < K * sum(tokens)
