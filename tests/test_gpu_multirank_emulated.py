"""G-rank expert parallelism emulated on ONE B200 (the pool has one GPU per call).

G contexts (ranks 0..G-1, MOE_EXCHANGE_EXTERNAL) share the device.  The staged
C-ABI runs exactly the device code of the NCCL path — gate, exchange plan,
dispatch into the local receive buffer AND the send buffer (row codes with the
remote bit), grouped GEMMs over received segments, combine from local rows AND
the return buffer — while the test moves the chunks between the ranks'
buffers with device-to-device copies in the same (peer, replica) order the
NCCL grouped send/recv uses.  Each rank's output must match the single-rank
oracle layer on its own tokens; ids and counts bit-exact.
"""
import numpy as np
import pytest

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import MOE_EXCHANGE_EXTERNAL, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


def _emulate(cuda, G, E, k, d, ff, tokens, rc, rg):
    import torch
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    ranks = []
    for r in range(G):
        m = MoELayer(1, E, k, d, ff, max_tokens=max(tokens), world_size=G, rank=r,
                     exchange_mode=MOE_EXCHANGE_EXTERNAL)
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
        m.set_placement(0, rc, rg)
        x = wl.tokens(tokens[r], d, E, 1, 50 + r)
        xd = torch.from_numpy(x.view(np.int16)).to(cuda)
        ranks.append(dict(m=m, x=x, xd=xd))
    for R in ranks:
        R["m"].begin(0, R["xd"])
        R["counts"] = R["m"].read_buffer(7, np.int32, (E,))
    counts_all = np.stack([R["counts"] for R in ranks]).astype(np.int32)
    for r, R in enumerate(ranks):
        R["m"].begin(0, R["xd"], counts_all)
        R["plan"] = pk.exchange_plan(G, r, counts_all, rc, rg)
    row_bytes = d * 2

    def move(src_which, dst_which, forward):
        for r, R in enumerate(ranks):
            chunks = R["plan"]["sends"] if forward else R["plan"]["recvs"]
            for (peer, f, off, n) in chunks:
                P = ranks[peer]
                peer_chunks = P["plan"]["recvs"] if forward else P["plan"]["sends"]
                dst_off = [c[2] for c in peer_chunks if c[0] == r and c[1] == f]
                assert len(dst_off) == 1 and [c[3] for c in peer_chunks if c[0] == r and c[1] == f][0] == n
                src_ptr, _ = R["m"].buffer(src_which)
                dst_ptr, _ = P["m"].buffer(dst_which)
                R["m"].memcpy(dst_ptr + dst_off[0] * row_bytes, src_ptr + off * row_bytes, n * row_bytes)

    move(1, 0, True)     # send X  -> peers' received rows
    for R in ranks:
        R["m"].expert(0)
    move(2, 3, False)    # expert Y -> owners' return buffers
    total_rows = 0
    for r, R in enumerate(ranks):
        T = tokens[r]
        yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
        R["m"].end(yd)
        y = oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))
        y_ref, ids_o, _, counts_o = oracle.layer_forward(R["x"], wg, experts, [1] * E, k)
        assert np.array_equal(R["counts"], counts_o)
        ids = R["m"].read_buffer(4, np.int32, (T, k))
        assert np.array_equal(ids, ids_o)
        err = row_rel_err(y, y_ref)
        assert err <= 2e-2, (r, err)
        total_rows += R["plan"]["rows_local"]
        R["m"].close()
    assert total_rows == k * sum(tokens)


@pytest.mark.parametrize("G,E,k,d,ff,tokens,rc,rg", [
    (2, 8, 2, 1024, 1408, [300, 170], [2, 1, 1, 3, 1, 1, 1, 1], [0, 1, 1, 0, 0, 1, 0, 1, 1, 0, 1]),
    (4, 8, 2, 1024, 1408, [64, 200, 1, 129], [1, 2, 1, 1, 1, 2, 1, 1], [0, 1, 2, 3, 0, 1, 2, 3, 0, 1]),
    (8, 16, 2, 1024, 1408, [33] * 8, [1] * 16, list(range(8)) * 2),
    (8, 64, 8, 2048, 1408, [32] * 8, [1] * 60 + [2, 3, 1, 2], [i % 8 for i in range(68)]),
])
def test_expert_parallel_emulated(cuda, G, E, k, d, ff, tokens, rc, rg):
    _emulate(cuda, G, E, k, d, ff, tokens, np.array(rc, np.int32), np.array(rg, np.int32))
