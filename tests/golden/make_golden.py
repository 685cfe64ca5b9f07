#!/usr/bin/env python
"""Generates the committed golden fixtures in tests/golden/.

  python tests/golden/make_golden.py

* route_loads.json — per-expert loads of the REFERENCE route_tokens
  (workload.cpp:188-230), produced by the compiled, unmodified reference
  (oracle/_ref/libmoeless_ref.so).  These pin the oracle's id replay and the
  product's routing restatement to the reference itself.
* planner.json — reference scale_experts / place_experts / layer_forward_time /
  predict outputs on seeded random instances (also from oracle/_ref).
* gate_small.npz, dispatch_small.npz, ffn_small.npz, layer_small.npz — outputs
  of the CPU oracle (oracle/moe_oracle.c) on small synthetic inputs.  The
  reference has no code for these, so they pin the oracle
  against regressions; GPU parity tests compare the device against the oracle.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

ROUTE_CASES = [
    # tokens, layer, iteration, experts, top_k, zipf_s, seed, drift
    (2048, 0, 0, 8, 2, 1.2, 1, 0),
    (16384, 1, 3, 8, 2, 1.2, 1, 0),
    (16384, 2, 5, 16, 2, 1.2, 1, 0),
    (256, 0, 1, 64, 8, 1.2, 1, 0),
    (256, 3, 7, 64, 8, 2.0, 1, 0),
    (400, 0, 3, 16, 2, 1.2, 99, 0),
    (50, 0, 0, 4, 4, 1.2, 1, 0),
    (1000, 1, 250, 8, 2, 1.2, 7, 100),
    (0, 0, 0, 8, 2, 1.2, 1, 0),
]


def ref_route(ref, c):
    T, layer, it, E, k, s, seed, drift = c
    loads = np.zeros(E, np.int64)
    rc = ref.ref_route_tokens(T, layer, it, E, 8, s, seed, k, drift, oracle.P(loads))
    assert rc == 0
    return loads.tolist()


def planner_cases(ref, n=300):
    rng = np.random.default_rng(2026)
    out = []
    for i in range(n):
        E = int(rng.integers(1, 13))
        loads = [int(v) if rng.random() > 0.2 else 0 for v in rng.integers(0, 1000, E)]
        mem = 1.0
        cap = float(rng.integers(0, 17))
        cv = float(rng.integers(0, 11)) / 10
        excl = int(rng.integers(0, 2))
        counts = np.zeros(E, np.int32)
        alloc = np.zeros(1)
        steps = np.zeros(1, np.int32)
        split = np.zeros(64, np.int32)
        cvt = np.zeros(64)
        ok = np.zeros(1, np.int32)
        la = np.asarray(loads, np.int64)
        assert ref.ref_scale_experts(oracle.P(la), E, 0, mem, cap, cv, excl, oracle.P(counts), oracle.P(alloc),
                                     oracle.P(steps), oracle.P(split), 64, oracle.P(cvt), oracle.P(ok)) == 0
        G = int(rng.integers(1, 6))
        reg = ref.ref_registry_new(3)
        gpu = np.zeros(int(counts.sum()), np.int32)
        warm = np.zeros(1, np.int32)
        cold = np.zeros(1, np.int32)
        assert ref.ref_place_experts(reg, oracle.P(la), oracle.P(counts), E, 0, mem, G, 1e9, i, 0, 0.0, 1.0,
                                     oracle.P(gpu), oracle.P(warm), oracle.P(cold)) == 0
        ref.ref_registry_free(reg)
        actual = rng.integers(0, 1000, E).astype(np.int64)
        out6 = np.zeros(6)
        assert ref.ref_layer_forward_time(oracle.P(la), oracle.P(counts), oracle.P(gpu), oracle.P(actual), E, G,
                                          0.01, 0.002, 0.5, 0.0, 330.0, oracle.P(out6)) == 0
        out.append(dict(loads=loads, cap=cap, cv=cv, excl=excl, counts=counts.tolist(), alloc=float(alloc[0]),
                        split=split[:int(steps[0])].tolist(), cv_trace=cvt[:min(int(steps[0]), 64)].tolist(),
                        verify_ok=int(ok[0]), G=G, gpu=gpu.tolist(), warm=int(warm[0]), cold=int(cold[0]),
                        actual=actual.tolist(), forward=out6.tolist()))
    return out


def main():
    ref = oracle.ref()
    if ref is None:
        raise SystemExit("oracle/_ref (compiled reference) is required to regenerate goldens")
    route = [dict(case=list(c), loads=ref_route(ref, c)) for c in ROUTE_CASES]
    json.dump(route, open(os.path.join(HERE, "route_loads.json"), "w"), indent=0)
    json.dump(planner_cases(ref), open(os.path.join(HERE, "planner.json"), "w"))

    # small synthetic layer (d=256, ff=256, E=8, k=2, T=64)
    E, k, d, ff, T = 8, 2, 256, 256, 64
    key_x = oracle.orc().orc_stream_key(1, 0, 0, 0x78746F6B)
    x = oracle.synth_tokens(key_x, 0, T, d, E)
    perm, w = oracle.popularity(E, 1.2, 1, 0)
    noise = np.array([3, 1, 7, 0, 5, 2, 6, 4], np.int32)
    wg = oracle.synth_gate(oracle.orc().orc_stream_key(1, 0, 0, 0x67617465), d, E, w, noise)
    ids, gw, counts, logits = oracle.gate(x, wg, k, want_logits=True)
    np.savez_compressed(os.path.join(HERE, "gate_small.npz"), x=x, wg=wg, ids=ids, w=gw, counts=counts,
                        logits=logits, pop_w=w, noise=noise)
    # dispatch over 2 ranks with replicas spread across them
    ids2 = [ids[:40], ids[40:]]
    rc = np.array([2, 1, 1, 3, 1, 1, 1, 1], np.int32)
    rg = np.array([0, 1, 1, 0, 0, 1, 0, 1, 1, 0, 1], np.int32)
    per, ss, sr, rows = oracle.dispatch(ids2, k, E, rc, rg)
    np.savez_compressed(os.path.join(HERE, "dispatch_small.npz"), ids0=ids2[0], ids1=ids2[1], rc=rc, rg=rg,
                        dg0=per[0][0], dr0=per[0][1], dg1=per[1][0], dr1=per[1][1], seg_start=ss, seg_rows=sr,
                        rows=rows)
    experts = [oracle.synth_expert(oracle.orc().orc_stream_key(1, 0, e, 0x65787074), d, ff) for e in range(E)]
    y_ffn = oracle.expert_ffn(x[:16], *experts[0], round_h=False, round_y=False)
    np.savez_compressed(os.path.join(HERE, "ffn_small.npz"), x=x[:16], w1=experts[0][0], w3=experts[0][1],
                        w2=experts[0][2], y=y_ffn)
    y, lids, lw, lcounts = oracle.layer_forward(x, wg, experts, [1, 2, 1, 1, 1, 1, 3, 1], k, round_h=True)
    np.savez_compressed(os.path.join(HERE, "layer_small.npz"), y=y, ids=lids, w=lw, counts=lcounts,
                        rc=np.array([1, 2, 1, 1, 1, 1, 3, 1], np.int32))
    print("goldens written to", HERE)


if __name__ == "__main__":
    main()
