"""C-ABI library loads and exports every declared symbol; the product's
synthetic-input generator and exchange plan agree with the oracle (CPU only,
no compute calls that need a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import _capi
from paper_2603_06350_b200 import workload as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "moe_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_capi.EXPORTED) == syms


def test_product_never_links_the_oracle():
    # the shipped library must not depend on oracle/ (test infrastructure)
    blob = open(_capi.LIB_PATH, "rb").read()
    assert b"libmoe_oracle" not in blob and b"libmoeless_ref" not in blob and b"orc_gate" not in blob


def test_ctx_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pk.MoeError):
        pk.MoELayer(1, 8, 2, 1024, 3584, max_tokens=16)


def test_ctx_desc_validation():
    for kw in [dict(num_experts=0), dict(top_k=3), dict(d_model=100), dict(d_ff=100), dict(max_tokens=0)]:
        args = dict(num_layers=1, num_experts=8, top_k=2, d_model=1024, d_ff=3584, max_tokens=16)
        args.update(kw)
        with pytest.raises(ValueError):
            pk.MoELayer(**args)


@pytest.mark.parametrize("T,d,E", [(17, 256, 8), (3, 2048, 64), (5, 4096, 16)])
def test_synth_matches_oracle(T, d, E):
    key = pk.stream_key(1, 2, 3, wl.TAG_TOKENS)
    assert np.array_equal(pk.synth_tokens(key, 10, T, d, E), oracle.synth_tokens(key, 10, T, d, E))
    _, w = pk.popularity(E, 4, 1.2, 1, 2)
    noise = wl.noise_permutation(E, 1, 2, 5)
    assert np.array_equal(pk.synth_gate(key, d, E, w, noise), oracle.synth_gate(key, d, E, w, noise))
    a = pk.synth_expert(key, d, 128)
    b = oracle.synth_expert(key, d, 128)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))


def test_synthetic_gate_grid_is_exact():
    """Every partial sum of x·Wg is a multiple of 2^-16 below 2^6 in magnitude:
    fp32 sums are exact in any order, so GPU and CPU ids agree bit for bit."""
    E, d, T = 16, 4096, 64
    x = oracle.bf16_to_f32(wl.tokens(T, d, E, 1, 0)).astype(np.float64)
    wg = oracle.bf16_to_f32(wl.gate_weights(E, d, 1.2, 1, 0, 0)).astype(np.float64)
    prods = x[:, None, :] * wg[None, :, :]
    assert np.all(prods * 65536 == np.round(prods * 65536))
    assert np.max(np.sum(np.abs(prods), axis=2)) < 64


def test_synthetic_routing_tracks_route_tokens_distribution():
    """Gumbel-top-k of log w is sampling without replacement ∝ w — the law of
    the reference's route_tokens (workload.cpp:188-230)."""
    E, k, d, T = 8, 2, 512, 8192
    x = wl.tokens(T, d, E, 1, 3)
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 3)
    _, _, counts = oracle.gate(x, wg, k)
    ref_loads = pk.route_tokens(T, 0, 3, E, 1, 1.2, 1, k)
    share = counts / counts.sum()
    ref_share = np.asarray(ref_loads) / np.sum(ref_loads)
    assert np.max(np.abs(share - ref_share)) < 0.02


def test_exchange_plan_matches_oracle_dispatch():
    rng = np.random.default_rng(11)
    for _ in range(60):
        G, E, k = int(rng.integers(1, 9)), int(rng.integers(2, 17)), 2
        ids = [np.stack([rng.permutation(E)[:k] for _ in range(int(rng.integers(1, 60)))]).astype(np.int32)
               for _ in range(G)]
        rc = rng.integers(1, 4, E).astype(np.int32)
        rg = rng.integers(0, G, int(rc.sum())).astype(np.int32)
        counts_all = np.stack([np.bincount(a.reshape(-1), minlength=E) for a in ids]).astype(np.int32)
        per, ss, sr, rows = oracle.dispatch(ids, k, E, rc, rg)
        for rank in range(G):
            p = pk.exchange_plan(G, rank, counts_all, rc, rg)
            assert p["rows_local"] == rows[rank]
            assert p["seg_rows"] == sr.tolist()
            for f in range(len(rg)):
                if rg[f] == rank:
                    assert p["seg_start"][f] == ss[f]
            # rows other ranks send me land exactly where the oracle puts them
            for (peer, f, off, n) in p["recvs"]:
                dg, dr = per[peer]
                mine = np.sort(dr[dg == rank])
                assert np.all(np.isin(np.arange(off, off + n), mine))
            sent = sum(n for (_, _, _, n) in p["sends"])
            assert sent == p["rows_send"] == int(np.sum(per[rank][0] != rank))


def test_oracle_generator_matches_product_generator():
    """bench.py's reference arm synthesises its inputs with the oracle's
    generator (oracle/workload.py) so it never loads the product; both must
    produce the same bytes as paper_2603_06350_b200/workload.py."""
    from oracle import workload as owl
    for (T, d, E, seed, batch) in [(64, 1024, 8, 1, 3), (33, 2048, 64, 1, 1001), (5, 4096, 16, 7, 0)]:
        assert np.array_equal(owl.tokens(T, d, E, seed, batch), wl.tokens(T, d, E, seed, batch))
    for (E, d, s, seed, layer, it) in [(8, 1024, 1.2, 1, 0, 5), (64, 2048, 2.0, 1, 0, 17), (16, 4096, 1.2, 3, 2, 0)]:
        assert np.array_equal(owl.gate_weights(E, d, s, seed, layer, it), wl.gate_weights(E, d, s, seed, layer, it))
    for a, b in zip(owl.expert_weights(1024, 256, 1, 0, 3), wl.expert_weights(1024, 256, 1, 0, 3)):
        assert np.array_equal(a, b)


def test_cpu_reference_layer_matches_oracle():
    """The CPU reference path of the bench (BLAS FFN) == the oracle layer (fp32)."""
    from oracle import workload as owl
    from oracle.cpu_path import CpuLayer
    E, k, d, ff, T = 8, 2, 1024, 512, 300
    ex = [owl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    x, wg = owl.tokens(T, d, E, 1, 0), owl.gate_weights(E, d, 1.2, 1, 0, 0)
    y, dt = CpuLayer(E, k, d, ff, ex).forward(x, wg)
    yr, _, _, _ = oracle.layer_forward(x, wg, ex, [1] * E, k, round_h=False)
    assert dt > 0
    assert float(np.max(np.abs(y - yr)) / np.max(np.abs(yr))) <= 1e-4
