"""CPU oracle — TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * oracle/libmoe_oracle.so   — the C restatement of the MoE data path
                                (oracle/moe_oracle.c; each function cites the
                                reference file:line it follows), and
  * oracle/_ref/libmoeless_ref.so — the UNMODIFIED reference simulator sources
                                compiled by oracle/Makefile (+ extern "C" shim).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmoe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoeless_ref.so")


def build(quiet: bool = True) -> None:
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        _orc = _load(ORACLE_SO)
        vp, i64, u64, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "orc_mix64": (u64, [u64]),
            "orc_keyed_draws": (None, [u64, u64, u64, u64, C.c_int, vp]),
            "orc_popularity_perm": (None, [C.c_int, u64, C.c_int, C.c_long, C.c_int, vp]),
            "orc_popularity_weights": (None, [C.c_int, dbl, vp, vp]),
            "orc_route_tokens_ids": (C.c_int, [i64, C.c_int, C.c_long, C.c_int, dbl, u64, C.c_int, C.c_int, vp, vp]),
            "orc_stream_key": (u64, [u64, u64, u64, u64]),
            "orc_synth_tokens": (None, [u64, i64, i64, C.c_int, C.c_int, vp]),
            "orc_synth_gate": (None, [u64, C.c_int, C.c_int, vp, vp, vp]),
            "orc_synth_expert": (None, [u64, C.c_int, C.c_int, vp, vp, vp]),
            "orc_gate": (None, [vp, i64, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, vp]),
            "orc_predict_mlp": (None, [vp, i64, C.c_int, vp, C.c_int, vp, C.c_int, vp]),
            "orc_dispatch": (C.c_int, [C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp]),
            "orc_expert_ffn": (None, [vp, i64, C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_int, vp]),
            "orc_combine": (None, [vp, C.c_int, vp, vp, i64, C.c_int, vp]),
            "orc_layer_forward": (C.c_int, [vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp,
                                            C.c_int, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_orc, name)
            f.restype, f.argtypes = res, args
    return _orc


def ref():
    """The compiled reference (None when it was never built and sources are absent)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            try:
                build()
            except Exception:
                return None
        if not os.path.exists(REF_SO):
            return None
        _ref = C.CDLL(REF_SO)
        vp, i64, u64, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_popularity_perm": (C.c_int, [C.c_int, C.c_int, dbl, u64, C.c_int, C.c_long, C.c_int, vp, vp]),
            "ref_route_tokens": (C.c_int, [i64, C.c_int, C.c_long, C.c_int, C.c_int, dbl, u64, C.c_int, C.c_int, vp]),
            "ref_scale_experts": (C.c_int, [vp, C.c_int, C.c_int, dbl, dbl, dbl, C.c_int, vp, vp, vp, vp, C.c_int,
                                            vp, vp]),
            "ref_registry_new": (vp, [C.c_int]),
            "ref_registry_free": (None, [vp]),
            "ref_registry_size": (C.c_long, [vp]),
            "ref_place_experts": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, dbl, C.c_int, dbl, C.c_long, C.c_int,
                                            dbl, dbl, vp, vp, vp]),
            "ref_update_registry": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_long]),
            "ref_layer_forward_time": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp]),
            "ref_predict": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, dbl,
                                      C.c_int, C.c_long, u64, vp, vp, vp]),
            "ref_measure_accuracy": (dbl, [vp, vp, C.c_int]),
            "ref_percentile": (dbl, [vp, C.c_int, dbl]),
            "ref_static_plan": (C.c_int, [vp, C.c_int, C.c_int, dbl, dbl, vp]),
            "ref_cpu_layer_path": (dbl, [i64, C.c_int, C.c_int, dbl, u64, C.c_int, dbl, dbl, C.c_int, vp]),
            "ref_gpu_comm_times": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, dbl, vp]),
            "ref_oracle_balance_time": (C.c_int, [vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp]),
            "ref_verify_plan": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, C.c_int, dbl, dbl, dbl, dbl,
                                          C.c_int, vp, C.c_char_p, C.c_int]),
            "ref_apply_finetuning": (C.c_int, [vp, C.c_int, dbl, vp]),
            "ref_coefficient_of_variation": (dbl, [vp, C.c_int]),
            "ref_serverful_cost": (dbl, [dbl, C.c_int, C.c_int, dbl, dbl]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_ref, name)
            f.restype, f.argtypes = res, args
    return _ref


def P(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# ----------------------------------------------------------- convenience
def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def route_ids(tokens, layer, iteration, experts, s, seed, top_k, drift=0):
    ids = np.zeros(tokens * top_k, np.int32)
    loads = np.zeros(experts, np.int64)
    rc = orc().orc_route_tokens_ids(tokens, layer, iteration, experts, s, seed, top_k, drift, P(ids), P(loads))
    assert rc == 0
    return ids.reshape(tokens, top_k), loads


def synth_tokens(key, first, tokens, d, experts):
    x = np.empty((tokens, d), np.uint16)
    orc().orc_synth_tokens(key, first, tokens, d, experts, P(x))
    return x


def synth_gate(key, d, experts, pop_w, noise_perm):
    wg = np.empty((experts, d), np.uint16)
    pw = np.ascontiguousarray(pop_w, np.float64)
    npm = np.ascontiguousarray(noise_perm, np.int32)
    orc().orc_synth_gate(key, d, experts, P(pw), P(npm), P(wg))
    return wg


def synth_expert(key, d, ff):
    w1 = np.empty((ff, d), np.uint16)
    w3 = np.empty((ff, d), np.uint16)
    w2 = np.empty((d, ff), np.uint16)
    orc().orc_synth_expert(key, d, ff, P(w1), P(w3), P(w2))
    return w1, w3, w2


def popularity(experts, s, seed, layer, iteration=0, drift=0):
    perm = np.zeros(experts, np.int32)
    w = np.zeros(experts, np.float64)
    orc().orc_popularity_perm(experts, seed, layer, iteration, drift, P(perm))
    orc().orc_popularity_weights(experts, s, P(perm), P(w))
    return perm, w


def gate(x, wg, top_k, want_logits=False):
    T, d = x.shape
    E = wg.shape[0]
    ids = np.zeros((T, top_k), np.int32)
    w = np.zeros((T, top_k), np.float32)
    counts = np.zeros(E, np.int32)
    logits = np.zeros((T, E), np.float32) if want_logits else None
    orc().orc_gate(P(np.ascontiguousarray(x)), T, d, P(np.ascontiguousarray(wg)), E, top_k, P(ids), P(w),
                   P(counts), P(logits) if want_logits else None)
    return (ids, w, counts, logits) if want_logits else (ids, w, counts)


def predict_mlp(x, w1, w2, top_k):
    """Histogram of top-k(W2 relu(W1 x)) per token (the MLP predictor)."""
    T, d = x.shape
    E = w1.shape[0]
    counts = np.zeros(E, np.int32)
    orc().orc_predict_mlp(P(np.ascontiguousarray(x)), T, d, P(np.ascontiguousarray(w1)), E,
                          P(np.ascontiguousarray(w2, np.float32)), top_k, P(counts))
    return counts


def dispatch(ids_per_rank, top_k, experts, replica_counts, replica_gpu):
    """Returns per rank (dest_gpu[T*k], dest_row[T*k]), seg_start, seg_rows, rows_on_gpu."""
    G = len(ids_per_rank)
    ids_c = [np.ascontiguousarray(np.asarray(i, np.int32).reshape(-1)) for i in ids_per_rank]
    tokens = np.array([len(i) // top_k for i in ids_c], np.int64)
    dg = [np.zeros(len(i), np.int32) for i in ids_c]
    dr = [np.zeros(len(i), np.int64) for i in ids_c]
    rc = np.ascontiguousarray(replica_counts, np.int32)
    rg = np.ascontiguousarray(replica_gpu, np.int32)
    R = int(rc.sum())
    ss, sr, rows = np.zeros(R, np.int64), np.zeros(R, np.int64), np.zeros(G, np.int64)
    arr = lambda lst: (C.c_void_p * G)(*[C.c_void_p(a.ctypes.data) for a in lst])
    rc_ = orc().orc_dispatch(G, arr(ids_c), P(tokens), top_k, experts, P(rc), P(rg), arr(dg), arr(dr), P(ss),
                             P(sr), P(rows))
    assert rc_ == 0
    return [(dg[s], dr[s]) for s in range(G)], ss, sr, rows


def expert_ffn(x, w1, w3, w2, round_h=True, round_y=True):
    rows, d = x.shape
    ff = w1.shape[0]
    y = np.zeros((rows, d), np.float32)
    if rows:
        orc().orc_expert_ffn(P(np.ascontiguousarray(x)), rows, d, ff, P(w1), P(w3), P(w2), int(round_h),
                             int(round_y), P(y))
    return y


def combine(Y, rows, w, tokens, top_k):
    d = Y.shape[1]
    y = np.zeros((tokens, d), np.float32)
    orc().orc_combine(P(np.ascontiguousarray(Y, np.float32)), d, P(np.ascontiguousarray(rows, np.int64)),
                      P(np.ascontiguousarray(w, np.float32)), tokens, top_k, P(y))
    return y


def layer_forward(x, wg, experts_w, replica_counts, top_k, round_h=True):
    """Whole layer on one rank: returns (y fp32 [T,d], ids, w, counts)."""
    T, d = x.shape
    E = wg.shape[0]
    ff = experts_w[0][0].shape[0]
    y = np.zeros((T, d), np.float32)
    ids = np.zeros((T, top_k), np.int32)
    w = np.zeros((T, top_k), np.float32)
    counts = np.zeros(E, np.int32)
    arr = lambda j: (C.c_void_p * E)(*[C.c_void_p(experts_w[e][j].ctypes.data) for e in range(E)])
    rc = np.ascontiguousarray(replica_counts, np.int32)
    r = orc().orc_layer_forward(P(np.ascontiguousarray(x)), T, d, ff, E, top_k, P(np.ascontiguousarray(wg)),
                                arr(0), arr(1), arr(2), P(rc), int(round_h), P(y), P(ids), P(w), P(counts))
    assert r == 0
    return y, ids, w, counts
