"""fp32 mode (north_star: outputs within 1e-4 of the fp32 reference).

Gate inputs stay on the exact synthetic grid (ids bit-exact); the expert
weights are genuinely fp32 (not bf16-representable), so the check exercises
the fp32 FFMA data path against a float64 torch reference and the fp32 oracle.
"""
import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu
TOL_FP32 = 1e-4


@pytest.mark.parametrize("E,k,d,ff,T,rc", [(8, 2, 512, 384, 300, [1, 2, 1, 1, 1, 1, 1, 3]),
                                           (16, 2, 256, 256, 129, [1] * 16),
                                           (64, 8, 256, 128, 64, [1] * 64)])
def test_fp32_mode_within_1e4(cuda, E, k, d, ff, T, rc):
    import torch
    rng = np.random.default_rng(3)
    x = oracle.bf16_to_f32(wl.tokens(T, d, E, 1, 0))
    wg = oracle.bf16_to_f32(wl.gate_weights(E, d, 1.2, 1, 0, 0))
    experts = [((rng.standard_normal((ff, d)) / np.sqrt(d)).astype(np.float32),
                (rng.standard_normal((ff, d)) / np.sqrt(d)).astype(np.float32),
                (rng.standard_normal((d, ff)) / np.sqrt(ff)).astype(np.float32)) for _ in range(E)]
    m = MoELayer(1, E, k, d, ff, max_tokens=T, precision=1)
    m.set_gate(0, np.ascontiguousarray(wg))
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    m.set_placement(0, rc, [0] * int(np.sum(rc)))
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(cuda)
    yd = torch.zeros((T, d), dtype=torch.float32, device=cuda)
    m.forward(0, xd, yd, MOE_PLAN_FIXED, 0)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    # routing: bit-exact against the oracle on the exact grid
    ids_o, w_o, counts_o = oracle.gate(oracle.f32_to_bf16(x), oracle.f32_to_bf16(wg), k)
    assert np.array_equal(m.read_buffer(4, np.int32, (T, k)), ids_o)
    # float64 reference of the whole layer
    xt = torch.from_numpy(x).double()
    ref = torch.zeros((T, d), dtype=torch.float64)
    wts = torch.from_numpy(w_o).double()
    for e, (w1, w3, w2) in enumerate(experts):
        rows, slot = np.nonzero(ids_o == e)
        if len(rows) == 0:
            continue
        a = xt[rows] @ torch.from_numpy(w1).double().T
        b = xt[rows] @ torch.from_numpy(w3).double().T
        h = a * torch.sigmoid(a) * b
        ref.index_add_(0, torch.from_numpy(rows), wts[rows, slot, None] * (h @ torch.from_numpy(w2).double().T))
    err = row_rel_err(y, ref.numpy())
    assert err <= TOL_FP32, err
    m.close()


def test_fp32_mode_two_ranks_peer_memory(cuda):
    """fp32 mode with two ranks sharing the GPU over the peer-memory exchange
    (SYNC planning: host-planned exchange, fp32 rows moved as opaque 16-byte
    chunks): each rank's output equals the single-GPU fp32 layer bit for bit."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from paper_2603_06350_b200 import MOE_EXCHANGE_P2P, MOE_PLAN_SYNC
    G, E, k, d, ff, T = 2, 8, 2, 256, 256, 96
    rng = np.random.default_rng(5)
    wg = oracle.bf16_to_f32(wl.gate_weights(E, d, 1.4, 1, 0, 0))
    experts = [((rng.standard_normal((ff, d)) / np.sqrt(d)).astype(np.float32),
                (rng.standard_normal((ff, d)) / np.sqrt(d)).astype(np.float32),
                (rng.standard_normal((d, ff)) / np.sqrt(ff)).astype(np.float32)) for _ in range(E)]
    mem = 3.0 * d * ff * 4 / 1e6
    ms = [MoELayer(1, E, k, d, ff, max_tokens=T, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P, precision=1,
                   expert_mem_mb=mem, layer_mem_cap_mb=(E + 2) * mem) for r in range(G)]
    handles = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(handles)
    one = MoELayer(1, E, k, d, ff, max_tokens=T, precision=1, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    for m in ms + [one]:
        m.set_gate(0, np.ascontiguousarray(wg))
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
    xs = [torch.from_numpy(np.ascontiguousarray(oracle.bf16_to_f32(wl.tokens(T, d, E, 1, 70 + r)))).to(cuda)
          for r in range(G)]
    ys = [torch.zeros((T, d), dtype=torch.float32, device=cuda) for _ in range(G)]
    with ThreadPoolExecutor(G) as ex:
        list(ex.map(lambda r: ms[r].forward(0, xs[r], ys[r], MOE_PLAN_SYNC, 0), range(G)))
    for m in ms:
        m.sync()
    for r in range(G):
        y1 = torch.zeros_like(ys[r])
        one.forward(0, xs[r], y1, MOE_PLAN_FIXED, 0)
        one.sync()
        assert torch.equal(ys[r], y1), r
    for m in ms + [one]:
        m.close()
