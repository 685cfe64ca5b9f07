"""Expert-parallel (N > 1) path on CPU: world_size 2 and 3 over gloo.

Each rank gates its own token shard, the ranks all-gather the per-expert
counts, every rank builds its exchange plan with the PRODUCT host code
(exchange_plan.cpp via the C-ABI), rows move between processes with
point-to-point send/recv exactly as the NCCL path issues them (one message
per (peer, replica) chunk, both sides in (peer, replica) order), the experts
run (oracle FFN on each received segment), rows travel back, and the combine
must reproduce the single-process oracle layer for every rank's tokens.
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
        x = wl.tokens(T, D, E, 1, 100 + rank)
        ids, w, counts = oracle.gate(x, wg, K)
        parts = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(counts.astype(np.int32)))
        counts_all = torch.stack(parts).numpy()
        plan = pk.exchange_plan(world, rank, counts_all, rc, rg)

        # integer split restated for the transport side of the test
        rep_base = np.concatenate([[0], np.cumsum(rc)])
        n = counts_all.sum(0)
        start = np.zeros(len(rg), np.int64)
        for e in range(E):
            q_, r_ = divmod(int(n[e]), int(rc[e]))
            for r in range(rc[e]):
                start[rep_base[e] + r] = r * q_ + min(r, r_)
        src_off = counts_all[:rank].sum(0)
        mine = {e: [(t, j) for t in range(T) for j in range(K) if ids[t, j] == e] for e in range(E)}

        def my_rows(f):  # this rank's assignments that replica f owns, in global order
            e = int(np.searchsorted(rep_base, f, side="right") - 1)
            lo = max(start[f], src_off[e])
            hi = min(start[f] + plan["seg_rows"][f], src_off[e] + counts_all[rank, e])
            return [mine[e][i] for i in range(int(lo - src_off[e]), int(hi - src_off[e]))], lo

        xp = np.zeros((plan["rows_local"], D), np.uint16)
        where = {}  # (t, j) -> ("local", row) | ("ret", row)
        for f in range(len(rg)):
            if rg[f] != rank:
                continue
            rows, lo = my_rows(f)
            for i, (t, j) in enumerate(rows):
                row = plan["seg_start"][f] + (lo - start[f]) + i
                xp[row] = x[t]
                where[(t, j)] = ("local", row)
        send = np.zeros((plan["rows_send"], D), np.uint16)
        for (peer, f, off, cnt) in plan["sends"]:
            rows, _ = my_rows(f)
            assert len(rows) == cnt
            for i, (t, j) in enumerate(rows):
                send[off + i] = x[t]
                where[(t, j)] = ("ret", off + i)
        assert len(where) == T * K

        def exchange(src_buf, src_chunks, dst_buf, dst_chunks):
            reqs = []
            bufs = []
            for (peer, f, off, cnt) in dst_chunks:
                b = torch.zeros((cnt, src_buf.shape[1]), dtype=torch.int16)
                bufs.append((b, off))
                reqs.append(dist.irecv(b, src=peer, tag=f))
            for (peer, f, off, cnt) in src_chunks:
                reqs.append(dist.isend(torch.from_numpy(src_buf[off:off + cnt].view(np.int16).copy()), dst=peer, tag=f))
            for r in reqs:
                r.wait()
            for b, off in bufs:
                dst_buf[off:off + b.shape[0]] = b.numpy().view(src_buf.dtype)

        exchange(send, plan["sends"], xp, plan["recvs"])  # dispatch all-to-all
        y_rows = np.zeros((plan["rows_local"], D), np.float32)
        for f in range(len(rg)):
            if rg[f] == rank and plan["seg_rows"][f] > 0:
                e = int(np.searchsorted(rep_base, f, side="right") - 1)
                s0, s1 = plan["seg_start"][f], plan["seg_start"][f] + plan["seg_rows"][f]
                y_rows[s0:s1] = oracle.expert_ffn(xp[s0:s1], *experts[e])
        yb = oracle.f32_to_bf16(y_rows)
        ret = np.zeros((plan["rows_send"], D), np.uint16)
        exchange(yb, plan["recvs"], ret, plan["sends"])  # combine all-to-all (reverse)
        y = np.zeros((T, D), np.float32)
        for t in range(T):
            for j in range(K):
                kind, row = where[(t, j)]
                src = yb if kind == "local" else ret
                y[t] += w[t, j] * oracle.bf16_to_f32(src[row])
        y_ref, ids_ref, _, _ = oracle.layer_forward(x, wg, experts, [1] * E, K)
        assert np.array_equal(ids, ids_ref)
        err = row_rel_err(y, y_ref)
        q.put((rank, err, plan["rows_local"], plan["rows_send"]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # surface the failure to the parent
        import traceback
        q.put((rank, "ERR " + traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("world,rc,rg,tokens", [
    (2, [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 0, 1, 0, 1, 1, 0, 1], [40, 33]),
    (2, [1] * 8, [0, 1, 0, 1, 0, 1, 0, 1], [24, 1]),
    (3, [3, 1, 2, 1, 1, 1, 1, 1], [0, 1, 2, 2, 0, 1, 1, 0, 2, 0, 1], [17, 30, 9]),
])
def test_expert_parallel_over_gloo(world, rc, rg, tokens):
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
    total_rows = 0
    for rank, err, rows_local, rows_send in res:
        assert not isinstance(err, str), err
        assert err <= 2e-2
        total_rows += rows_local
    assert total_rows == K * sum(tokens)
