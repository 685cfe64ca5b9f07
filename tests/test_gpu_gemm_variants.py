"""The K4 kernels — 1-SM (M=128 tiles), 2-SM cta_group::2 (M=256 tiles across
an SM pair), single-CTA M=256 (two MMAs sharing B) and swap-AB decode tiles
(weights as M, up to 64 tokens as N) — against the oracle and against each other, on ragged
segments (partial tiles, single-row segments, replicas co-located)."""
import os

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import MOE_PLAN_FIXED, MoELayer
from paper_2603_06350_b200 import workload as wl
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


def _run(cuda, variant, E, k, d, ff, T, rc, seed=21, env=None):
    import torch
    env = dict(env or {}, MOE_GEMM_VARIANT=variant)
    os.environ.update(env)
    try:
        m = MoELayer(1, E, k, d, ff, max_tokens=T)
    finally:
        for key in env:
            del os.environ[key]
    x = wl.tokens(T, d, E, seed, 0)
    wg = wl.gate_weights(E, d, 1.2, seed, 0, 0)
    experts = [wl.expert_weights(d, ff, seed, 0, e) for e in range(E)]
    m.set_gate(0, wg)
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    m.set_placement(0, rc, [0] * int(np.sum(rc)))
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
    m.forward(0, xd, yd, MOE_PLAN_FIXED, 0)
    torch.cuda.synchronize()
    m.close()
    return x, wg, experts, oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16))


@pytest.mark.parametrize("E,k,d,ff,T,rc", [
    (8, 2, 1024, 1408, 2048, [1, 2, 1, 1, 3, 1, 1, 1]),
    (8, 2, 2048, 3584, 700, [1] * 8),
    (16, 2, 1024, 1408, 1500, [2] * 16),
    (4, 1, 256, 128, 5, [1] * 4),
    (64, 8, 2048, 1408, 256, [2] + [1] * 62 + [3]),   # cfg5 decode shape
    (8, 2, 1024, 1408, 200, [1, 1, 2, 1, 1, 1, 1, 1]),  # 33-64-row and >64-row segments
])
def test_variants_agree_and_match_oracle(cuda, E, k, d, ff, T, rc):
    x, wg, experts, y1 = _run(cuda, "1sm", E, k, d, ff, T, rc)
    _, _, _, y2 = _run(cuda, "2sm", E, k, d, ff, T, rc)
    _, _, _, y3 = _run(cuda, "m256", E, k, d, ff, T, rc)
    _, _, _, y4 = _run(cuda, "swap", E, k, d, ff, T, rc)  # GEMM1 + GEMM2 in one launch
    _, _, _, y5 = _run(cuda, "swap", E, k, d, ff, T, rc, env={"MOE_SWAP_FUSE": "0"})
    _, _, _, y6 = _run(cuda, "swap64", E, k, d, ff, T, rc)
    _, _, _, y7 = _run(cuda, "swap128", E, k, d, ff, T, rc)
    _, _, _, y8 = _run(cuda, "mc", E, k, d, ff, T, rc)  # cluster pairs, B multicast
    _, _, _, y9 = _run(cuda, "2sm", E, k, d, ff, T, rc, env={"MOE_GEMM_SCHED": "dynamic"})  # claimed tiles
    y_ref = oracle.layer_forward(x, wg, experts, rc, k)[0]
    for y in (y1, y2, y3, y4, y5, y6, y7, y8, y9):
        err = row_rel_err(y, y_ref)
        assert err <= 2e-2, err
    # same K order per output element, same fp32 accumulation: bit-identical outputs
    assert np.array_equal(y1, y2) and np.array_equal(y1, y3)
    # swap-AB (weights as M, tokens as N): the same products in the same K order
    assert np.array_equal(y1, y4), float(np.max(np.abs(y1 - y4)))
    assert np.array_equal(y1, y5), float(np.max(np.abs(y1 - y5)))
    assert np.array_equal(y1, y6) and np.array_equal(y1, y7)
    assert np.array_equal(y1, y8)  # multicast B: the same MMAs on the same operands
    assert np.array_equal(y1, y9)  # tile order does not change any tile's arithmetic


def test_swap_fused_repeated_forwards(cuda):
    """The fused swap-AB launch resets its readiness counters itself: many
    forwards in a row (eager and CUDA-graph replay) stay equal to the 1-SM
    kernel's output."""
    import torch
    E, k, d, ff, T = 64, 8, 1024, 1408, 128
    x, wg, experts, y1 = _run(cuda, "1sm", E, k, d, ff, T, [1] * E)
    for graphs in (False, True):
        m = MoELayer(1, E, k, d, ff, max_tokens=T, cuda_graphs=graphs)
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
        xd = torch.from_numpy(x.view(np.int16)).to(cuda)
        for it in range(20):
            yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
            m.forward(0, xd, yd, MOE_PLAN_FIXED, it)
            m.sync()
            assert np.array_equal(oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16)), y1), (graphs, it)
        m.close()


@pytest.mark.timeout(300)
def test_swap_fused_concurrent_contexts(cuda):
    """Two contexts on one GPU running fused swap-AB forwards at the same time
    from two host threads (their persistent grids compete for the SMs): the
    claimed-tile schedule must neither deadlock nor change a bit."""
    import threading

    import torch
    E, k, d, ff, T = 64, 8, 1024, 1408, 256
    x, wg, experts, y1 = _run(cuda, "1sm", E, k, d, ff, T, [1] * E)
    layers = []
    for _ in range(2):
        m = MoELayer(1, E, k, d, ff, max_tokens=T)
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
        layers.append(m)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    outs = [[None] * 30 for _ in layers]
    errors = []

    def worker(i):
        try:
            torch.cuda.set_device(cuda)
            for it in range(30):
                yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
                layers[i].forward(0, xd, yd, MOE_PLAN_FIXED, it)
                layers[i].sync()
                outs[i][it] = yd.cpu().numpy()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(2):
        for it in range(30):
            assert np.array_equal(oracle.bf16_to_f32(outs[i][it].view(np.uint16)), y1), (i, it)
    for m in layers:
        m.close()


@pytest.mark.parametrize("mask", ["0", "15"])
@pytest.mark.parametrize("graphs", [False, True])
def test_pdl_front_masks_bit_identical(cuda, mask, graphs):
    """Programmatic launches of the block prefix / dispatch / combine
    (MOE_PDL_FRONT) change only scheduling: outputs equal the default's."""
    import torch
    E, k, d, ff, T = 16, 2, 1024, 1408, 700
    x, wg, experts, y_ref = _run(cuda, "1sm", E, k, d, ff, T, [1] * E)
    os.environ["MOE_PDL_FRONT"] = mask
    try:
        m = MoELayer(1, E, k, d, ff, max_tokens=T, cuda_graphs=graphs)
    finally:
        del os.environ["MOE_PDL_FRONT"]
    m.set_gate(0, wg)
    for e, w in enumerate(experts):
        m.load_expert(0, e, *w)
    xd = torch.from_numpy(x.view(np.int16)).to(cuda)
    for it in range(3):
        yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
        m.forward(0, xd, yd, MOE_PLAN_FIXED, it)
        m.sync()
        assert np.array_equal(oracle.bf16_to_f32(yd.cpu().numpy().view(np.uint16)), y_ref), (mask, graphs, it)
    m.close()
