"""paper_2603_06350_b200 — B200-native MoE-layer data path for MoEless (arXiv 2603.06350).

Host-side mirror of the reference interface for this path
(/root/reference/proj/include/moeless/*.hpp) over the C-ABI library
libmoe_b200.so (include/moe_b200.h):

  planner (host C++):  scale_experts, place_experts, ReplicaRegistry,
                       update_registry, layer_forward_time (analytic model),
                       predict, measure_accuracy, route_tokens, percentile
  data path (sm_100a): MoELayer.forward  = gate -> replica-aware dispatch ->
                       SwiGLU grouped GEMM (tcgen05) -> combine [-> NCCL EP]

Names, argument meaning and error behaviour follow the reference: bad input
raises ValueError (std::invalid_argument), infeasible placement raises
MoeError (std::runtime_error) with the reference wording.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import (MOE_EXCHANGE_COPY, MOE_EXCHANGE_EXTERNAL, MOE_EXCHANGE_NCCL, MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MOE_PLAN_PREDICTED,
                    MOE_PLAN_SYNC, MoeChunk, MoeCtxDesc, MoeError, MoeLayerStats, MoeP2PHandle, check, lib)

__all__ = [
    "scale_experts", "place_experts", "ReplicaRegistry", "update_registry", "layer_forward_time",
    "predict", "measure_accuracy", "route_tokens", "popularity", "percentile", "exchange_plan",
    "exchange_plan_direct",
    "MoELayer", "ScalingPlan", "PlaceResult", "synth_tokens", "synth_gate", "synth_expert",
    "stream_key", "nccl_unique_id", "PinnedArray", "MoeError", "MOE_PLAN_FIXED", "MOE_PLAN_SYNC",
    "MOE_PLAN_PREDICTED", "MOE_EXCHANGE_NCCL",
    "MOE_EXCHANGE_EXTERNAL", "MOE_EXCHANGE_P2P", "MOE_EXCHANGE_COPY", "LIB_PATH",
]
LIB_PATH = _capi.LIB_PATH


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _i64(v: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64))


def _i32(v: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int32))


# ------------------------------------------------------------------ planner
@dataclass
class ScalingPlan:
    """reference types.hpp:49-69 (shares are loads[e]/replica_counts[e])."""
    layer: int
    replica_counts: List[int]
    loads: List[int]
    alloc_mem_mb: float
    expert_mem_mb: float
    split_trace: List[int] = field(default_factory=list)
    cv_trace: List[float] = field(default_factory=list)

    def total_replicas(self) -> int:
        return int(sum(self.replica_counts))


def scale_experts(loads: Sequence[int], expert_mem_mb: float, layer_mem_cap_mb: float,
                  cv_threshold: float = 0.2, exclude_zero_loads_from_cv: bool = False,
                  layer: int = 0) -> ScalingPlan:
    """Algorithm 1 (reference scaler.cpp:55-97)."""
    lv = _i64(loads)
    E = len(lv)
    counts = np.zeros(max(E, 1), np.int32)
    alloc = C.c_double()
    steps = C.c_int()
    cap = 4096
    split = np.zeros(cap, np.int32)
    cvt = np.zeros(cap, np.float64)
    check(lib.moe_plan_scale(_p(lv), E, layer, expert_mem_mb, layer_mem_cap_mb, cv_threshold,
                             int(exclude_zero_loads_from_cv), _p(counts), C.byref(alloc),
                             C.byref(steps), _p(split), _p(cvt), cap))
    n = min(steps.value, cap)
    return ScalingPlan(layer, counts[:E].tolist(), lv.tolist(), alloc.value, expert_mem_mb,
                       split[:n].tolist(), cvt[:n].tolist())


class ReplicaRegistry:
    """Keep-alive registry (reference placer.hpp:37-66)."""

    def __init__(self, keep_alive_iters: int = 0):
        h = C.c_void_p()
        check(lib.moe_registry_create(int(keep_alive_iters), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.moe_registry_destroy(self._h)
            self._h = None

    def size(self) -> int:
        return int(lib.moe_registry_size(self._h))


@dataclass
class PlaceResult:
    gpu_for: List[List[int]]
    warm_count: int
    cold_count: int

    def flat(self) -> List[int]:
        return [g for per in self.gpu_for for g in per]


def place_experts(plan: ScalingPlan, gpu_count: int, gpu_mem_capacity_mb: float,
                  registry: ReplicaRegistry, iteration: int, load_includes_compute: bool = False,
                  alpha_ms_per_token: float = 0.0, beta_ms_per_token: float = 1.0) -> PlaceResult:
    """Algorithm 2 (reference placer.cpp:45-122)."""
    lv, rc = _i64(plan.loads), _i32(plan.replica_counts)
    out = np.zeros(max(int(rc.sum()), 1), np.int32)
    warm, cold = C.c_int(), C.c_int()
    check(lib.moe_plan_place(registry._h, _p(lv), _p(rc), len(rc), plan.layer, plan.expert_mem_mb,
                             gpu_count, gpu_mem_capacity_mb, iteration, int(load_includes_compute),
                             alpha_ms_per_token, beta_ms_per_token, _p(out), C.byref(warm),
                             C.byref(cold)))
    gpu_for, i = [], 0
    for r in rc:
        gpu_for.append(out[i:i + r].tolist())
        i += int(r)
    return PlaceResult(gpu_for, warm.value, cold.value)


def update_registry(registry: ReplicaRegistry, replica_counts: Sequence[int],
                    gpu_flat: Sequence[int], gpu_count: int, layer: int, iteration: int) -> None:
    rc, g = _i32(replica_counts), _i32(gpu_flat)
    check(lib.moe_registry_update(registry._h, _p(rc), _p(g), len(rc), gpu_count, layer, iteration))


def layer_forward_time(plan_loads, replica_counts, gpu_flat, actual, gpu_count, alpha, beta,
                       t_misc, m_misc, expert_mem_mb) -> Tuple[float, ...]:
    """Analytic forward model (reference cost_model.cpp:91-122)."""
    out = np.zeros(6, np.float64)
    lv, rc, g, a = _i64(plan_loads), _i32(replica_counts), _i32(gpu_flat), _i64(actual)
    check(lib.moe_model_forward_time(_p(lv), _p(rc), _p(g), _p(a), len(rc), gpu_count, alpha,
                                     beta, t_misc, m_misc, expert_mem_mb, _p(out)))
    return tuple(out.tolist())


def static_plan(loads: Sequence[int], gpu_count: int, expert_mem_mb: float,
                gpu_mem_capacity_mb: float = 180000.0) -> List[int]:
    """Fixed placement, expert e -> GPU e mod G (reference baselines.cpp:32-60)."""
    lv = _i64(loads)
    out = np.zeros(max(len(lv), 1), np.int32)
    check(lib.moe_static_plan(_p(lv), len(lv), gpu_count, expert_mem_mb, gpu_mem_capacity_mb, _p(out)))
    return out[:len(lv)].tolist()


def round_robin_placement(replica_counts: Sequence[int], gpu_count: int, expert_mem_mb: float,
                          gpu_mem_capacity_mb: float = 180000.0) -> List[int]:
    """Replica f -> GPU f mod G, flattened (reference simulator.cpp:32-50)."""
    rc = _i32(replica_counts)
    out = np.zeros(max(int(rc.sum()), 1), np.int32)
    check(lib.moe_round_robin_placement(_p(rc), len(rc), gpu_count, expert_mem_mb, gpu_mem_capacity_mb,
                                        _p(out)))
    return out[:int(rc.sum())].tolist()


def gpu_comm_times(plan_loads, replica_counts, gpu_flat, gpu_count: int, beta: float) -> List[float]:
    """beta x shares hosted per GPU (reference cost_model.cpp:67-89)."""
    lv, rc, g = _i64(plan_loads), _i32(replica_counts), _i32(gpu_flat)
    out = np.zeros(gpu_count, np.float64)
    check(lib.moe_gpu_comm_times(_p(lv), _p(rc), _p(g), len(rc), gpu_count, beta, _p(out)))
    return out.tolist()


def oracle_balance_time(actual, gpu_count, alpha, beta, t_misc, m_misc, expert_mem_mb) -> Tuple[float, ...]:
    """Perfect-balance line (reference baselines.cpp:141-154): compute, comm, forward, replicas, mem, cost."""
    a = _i64(actual)
    out = np.zeros(6, np.float64)
    check(lib.moe_oracle_balance_time(_p(a), len(a), gpu_count, alpha, beta, t_misc, m_misc, expert_mem_mb,
                                      _p(out)))
    return tuple(out.tolist())


def verify_plan(loads, replica_counts, shares, alloc_mem_mb, expert_mem_mb, layer_mem_cap_mb,
                cv_threshold=0.2, exclude_zero=False) -> Tuple[bool, List[str]]:
    """verify_plan (reference scaler.cpp:99-173); shares = [(expert, ordinal, num, den)]."""
    lv, rc = _i64(loads), _i32(replica_counts)
    sh = np.asarray(shares, np.int64).reshape(-1, 4) if len(shares) else np.zeros((0, 4), np.int64)
    se, so = _i32(sh[:, 0]), _i32(sh[:, 1])
    sn, sd = _i64(sh[:, 2]), _i64(sh[:, 3])
    ok = C.c_int()
    buf = C.create_string_buffer(1 << 16)
    check(lib.moe_verify_plan(_p(lv), len(lv), _p(rc) if len(rc) else None, len(rc), _p(se), _p(so), _p(sn),
                              _p(sd), len(sh), alloc_mem_mb, expert_mem_mb, layer_mem_cap_mb, cv_threshold,
                              int(exclude_zero), C.byref(ok), buf, len(buf)))
    return bool(ok.value), [m for m in buf.value.decode().split("\n") if m]


def apply_finetuning(per_layer_accuracy, threshold: float) -> Tuple[List[float], List[bool]]:
    """apply_layer_aware_finetuning (reference predictor.cpp:188-199) on a noisy profile."""
    acc = np.ascontiguousarray(np.asarray(per_layer_accuracy, np.float64)).copy()
    ft = np.zeros(max(len(acc), 1), np.int32)
    check(lib.moe_apply_finetuning(_p(acc), len(acc), threshold, _p(ft)))
    return acc.tolist(), [bool(v) for v in ft[:len(acc)]]


def coefficient_of_variation(values) -> float:
    v = np.ascontiguousarray(np.asarray(values, np.float64))
    r = lib.moe_coefficient_of_variation(_p(v) if len(v) else None, len(v))
    if r < 0:
        raise ValueError(lib.moe_last_error().decode())
    return r


def serverful_cost(total_ms, num_layers, experts, expert_mem_mb, m_misc_mb=0.0) -> float:
    return lib.moe_serverful_cost(total_ms, num_layers, experts, expert_mem_mb, m_misc_mb)


def predict(kind: int, actual: Sequence[int], layer: int = 0, history=(), accuracy=None,
            distance: int = 1, decay: float = 0.04, window: int = 8, iteration: int = 0,
            seed: int = 1, popularity=None) -> Tuple[List[int], bool]:
    """reference predictor.cpp:146-166; kind 0 oracle, 1 noisy, 2 historical."""
    a = _i64(actual)
    E = len(a)
    hist = _i64(np.asarray(history, dtype=np.int64).reshape(-1)) if len(history) else np.zeros(1, np.int64)
    acc = np.ascontiguousarray(np.asarray(accuracy, np.float64)) if accuracy is not None else None
    pop = np.ascontiguousarray(np.asarray(popularity, np.float64)) if popularity is not None else None
    out = np.zeros(max(E, 1), np.int64)
    fb = C.c_int()
    check(lib.moe_plan_predict(kind, _p(a), E, layer, _p(hist), len(history),
                               _p(acc) if acc is not None else None,
                               len(acc) if acc is not None else 0, distance, decay, window,
                               iteration, seed, _p(pop) if pop is not None else None, _p(out),
                               C.byref(fb)))
    return out[:E].tolist(), bool(fb.value)


def measure_accuracy(predicted: Sequence[int], actual: Sequence[int]) -> float:
    p, a = _i64(predicted), _i64(actual)
    if len(p) != len(a):
        raise ValueError("vectors differ in expert count")
    v = lib.moe_measure_accuracy(_p(p), _p(a), len(a))
    if v < 0:
        raise ValueError(lib.moe_last_error().decode())
    return v


def percentile(values: Sequence[float], q: float) -> float:
    v = np.ascontiguousarray(np.asarray(values, np.float64))
    r = lib.moe_percentile(_p(v) if len(v) else None, len(v), q)
    if r < 0 and (len(v) == 0 or q < 0 or q > 1):
        raise ValueError(lib.moe_last_error().decode())
    return r


def route_tokens(tokens: int, layer: int, iteration: int, experts: int, layers: int,
                 zipf_s: float, seed: int, top_k: int, drift_period: int = 0) -> List[int]:
    """The reference's routing stand-in (workload.cpp:188-230), host C++."""
    out = np.zeros(experts, np.int64)
    check(lib.moe_route_tokens(tokens, layer, iteration, experts, layers, zipf_s, seed, top_k,
                               drift_period, _p(out)))
    return out.tolist()


def popularity(experts: int, layers: int, zipf_s: float, seed: int, layer: int, iteration: int = 0,
               drift_period: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    perm = np.zeros(experts, np.int32)
    w = np.zeros(experts, np.float64)
    check(lib.moe_popularity(experts, layers, zipf_s, seed, layer, iteration, drift_period,
                             _p(perm), _p(w)))
    return perm, w


def exchange_plan(world_size: int, rank: int, counts_all: np.ndarray,
                  replica_counts: Sequence[int], replica_gpu: Sequence[int]):
    """Integer replica split + row exchange chunks for `rank` (exchange_plan.cpp)."""
    ca = np.ascontiguousarray(np.asarray(counts_all, np.int32).reshape(world_size, -1))
    E = ca.shape[1]
    rc, rg = _i32(replica_counts), _i32(replica_gpu)
    R = int(rc.sum())
    cap = max(1, R * world_size)
    sends, recvs = (MoeChunk * cap)(), (MoeChunk * cap)()
    ns, nr = C.c_int(), C.c_int()
    rl, rs = C.c_int64(), C.c_int64()
    ss, sr = np.zeros(max(R, 1), np.int64), np.zeros(max(R, 1), np.int64)
    check(lib.moe_exchange_plan(world_size, rank, E, _p(ca), _p(rc), _p(rg), sends, C.byref(ns),
                                recvs, C.byref(nr), cap, C.byref(rl), C.byref(rs), _p(ss), _p(sr)))
    conv = lambda arr, n: [(c.peer, c.replica, c.row_offset, c.rows) for c in arr[:n]]
    return dict(sends=conv(sends, ns.value), recvs=conv(recvs, nr.value), rows_local=rl.value,
                rows_send=rs.value, seg_start=ss[:R].tolist(), seg_rows=sr[:R].tolist())


def exchange_plan_direct(world_size: int, rank: int, counts_all: np.ndarray,
                         replica_counts: Sequence[int], replica_gpu: Sequence[int]):
    """Peer-memory form of the plan: per replica, the destination rank and the
    row base in THAT rank's received-rows buffer (exchange_plan.cpp, direct)."""
    ca = np.ascontiguousarray(np.asarray(counts_all, np.int32).reshape(world_size, -1))
    E = ca.shape[1]
    rc, rg = _i32(replica_counts), _i32(replica_gpu)
    R = int(rc.sum())
    tgt, base = np.zeros(max(R, 1), np.int32), np.zeros(max(R, 1), np.int32)
    rl, rs = C.c_int64(), C.c_int64()
    check(lib.moe_exchange_plan_direct(world_size, rank, E, _p(ca), _p(rc), _p(rg), _p(tgt), _p(base),
                                       C.byref(rl), C.byref(rs)))
    return dict(rep_target=tgt[:R].tolist(), rep_row_base=base[:R].tolist(), rows_local=rl.value,
                rows_send=rs.value)


# ------------------------------------------------------- synthetic inputs
class PinnedArray:
    """numpy view of a page-locked host buffer from the library's allocator."""

    def __init__(self, shape, dtype):
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(lib.moe_host_alloc(max(nbytes, 16), C.byref(p)))
        self._p = p
        buf = (C.c_uint8 * max(nbytes, 16)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        if getattr(self, "_p", None):
            lib.moe_host_free(self._p)
            self._p = None


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.moe_nccl_unique_id(buf))
    return buf.raw

def stream_key(seed: int, a: int, b: int, tag: int) -> int:
    return int(lib.moe_stream_key(seed, a, b, tag))


def synth_tokens(key: int, first: int, tokens: int, d_model: int, experts: int,
                 out: Optional[np.ndarray] = None) -> np.ndarray:
    x = out if out is not None else np.empty((tokens, d_model), np.uint16)
    check(lib.moe_synth_tokens(key, first, tokens, d_model, experts, _p(x)))
    return x


def synth_gate(key: int, d_model: int, experts: int, pop_weights, noise_perm) -> np.ndarray:
    pw = np.ascontiguousarray(np.asarray(pop_weights, np.float64))
    npm = _i32(noise_perm)
    wg = np.empty((experts, d_model), np.uint16)
    check(lib.moe_synth_gate(key, d_model, experts, _p(pw), _p(npm), _p(wg)))
    return wg


def synth_expert(key: int, d_model: int, d_ff: int):
    w1 = np.empty((d_ff, d_model), np.uint16)
    w3 = np.empty((d_ff, d_model), np.uint16)
    w2 = np.empty((d_model, d_ff), np.uint16)
    check(lib.moe_synth_expert(key, d_model, d_ff, _p(w1), _p(w3), _p(w2)))
    return w1, w3, w2


# ---------------------------------------------------------------- the layer
class MoELayer:
    """One rank's view of an MoE layer stack on one B200 (libmoe_b200 context).

    Tensors passed to the device entry points are torch CUDA tensors (torch is
    used only as an allocator/stream provider); weights are host numpy uint16
    (bf16 bit patterns) in nn.Linear layout.
    """

    def __init__(self, num_layers: int, num_experts: int, top_k: int, d_model: int, d_ff: int,
                 max_tokens: int, world_size: int = 1, rank: int = 0, device: int = 0,
                 exchange_mode: int = MOE_EXCHANGE_NCCL, nccl_unique_id: Optional[bytes] = None,
                 num_predictor_targets: int = 0, expert_mem_mb: float = 0.0,
                 layer_mem_cap_mb: float = 0.0, gpu_mem_capacity_mb: float = 180000.0,
                 cv_threshold: float = 0.2, keep_alive_iters: int = 50, predictor_distance: int = 1,
                 precision: int = 0, cuda_graphs: bool = False, residency: int = 0, replica_slots: int = 0):
        d = MoeCtxDesc()
        d.num_layers, d.num_experts, d.top_k = num_layers, num_experts, top_k
        d.d_model, d.d_ff, d.max_tokens = d_model, d_ff, max_tokens
        d.world_size, d.rank, d.device, d.exchange_mode = world_size, rank, device, exchange_mode
        self._uid = C.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id else None
        d.nccl_unique_id = C.cast(self._uid, C.c_void_p) if self._uid is not None else None
        d.num_predictor_targets = num_predictor_targets
        d.expert_mem_mb = expert_mem_mb or 3.0 * d_model * d_ff * 2 / 1e6
        d.layer_mem_cap_mb, d.gpu_mem_capacity_mb = layer_mem_cap_mb, gpu_mem_capacity_mb
        d.cv_threshold, d.keep_alive_iters = cv_threshold, keep_alive_iters
        d.predictor_distance = predictor_distance
        d.precision = precision
        d.use_cuda_graphs = int(cuda_graphs)
        d.residency, d.replica_slots = residency, replica_slots
        self.fp32 = precision == 1
        h = C.c_void_p()
        check(lib.moe_ctx_create(C.byref(d), C.byref(h)))
        self._h = h
        self.desc = d
        self.E, self.k, self.d, self.ff = num_experts, top_k, d_model, d_ff
        self.world_size, self.rank = world_size, rank

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(lib.moe_ctx_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        s = C.c_void_p()
        check(lib.moe_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        check(lib.moe_ctx_sync(self._h))

    def residency(self, layer: int) -> Tuple[np.ndarray, int]:
        """(slot of each expert on this rank, -1 = not resident; slots in the layer's pool)."""
        out = np.empty(self.E, np.int32)
        n = C.c_int()
        check(lib.moe_residency(self._h, layer, out.ctypes.data, C.byref(n)))
        return out, n.value

    def p2p_export(self) -> bytes:
        """This rank's peer-memory handle (MOE_EXCHANGE_P2P): 192 opaque bytes
        to all-gather over any transport."""
        h = MoeP2PHandle()
        check(lib.moe_p2p_export(self._h, C.byref(h)))
        return C.string_at(C.addressof(h), C.sizeof(h))

    def p2p_import(self, handles: Sequence[bytes]) -> None:
        """Map every rank's slab (handles indexed by rank, this rank's included)."""
        arr = (MoeP2PHandle * len(handles))()
        for i, b in enumerate(handles):
            assert len(b) == C.sizeof(MoeP2PHandle)
            C.memmove(C.addressof(arr[i]), b, len(b))
        check(lib.moe_p2p_import(self._h, arr, len(handles)))

    def load_expert(self, layer: int, expert: int, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray):
        dt = np.float32 if self.fp32 else np.uint16
        for w, shape in ((w1, (self.ff, self.d)), (w3, (self.ff, self.d)), (w2, (self.d, self.ff))):
            if w.dtype != dt or w.shape != shape or not w.flags.c_contiguous:
                raise ValueError(f"expert weight must be C-contiguous {np.dtype(dt).name} {shape}")
        fn = lib.moe_load_expert_weights_f32 if self.fp32 else lib.moe_load_expert_weights
        check(fn(self._h, layer, expert, _p(w1), _p(w3), _p(w2)))

    def set_gate(self, layer: int, wg: np.ndarray) -> None:
        dt = np.float32 if self.fp32 else np.uint16
        if wg.dtype != dt or wg.shape != (self.E, self.d) or not wg.flags.c_contiguous:
            raise ValueError(f"gate weight must be C-contiguous {np.dtype(dt).name} [E, d_model]")
        fn = lib.moe_set_gate_weights_f32 if self.fp32 else lib.moe_set_gate_weights
        check(fn(self._h, layer, _p(wg)))

    def set_gate_device(self, layer: int, wg) -> None:
        """Gate weights from a device tensor ([E, d_model], the context's precision),
        stream-ordered on the context's stream."""
        if tuple(wg.shape) != (self.E, self.d) or not wg.is_contiguous():
            raise ValueError("gate weight must be a contiguous [E, d_model] device tensor")
        check(lib.moe_set_gate_weights_device(self._h, layer, C.c_void_p(wg.data_ptr()), None))

    def set_predictor(self, layer: int, slot: int, wp: np.ndarray) -> None:
        check(lib.moe_set_predictor_weights(self._h, layer, slot, _p(np.ascontiguousarray(wp))))

    def set_predictor_mlp(self, layer: int, slot: int, w1, w2) -> None:
        """MLP predictor for `slot`: w1 [E, d] bf16 bits (None keeps the rows),
        w2 [E, E] fp32 (None: back to linear)."""
        a1 = None if w1 is None else np.ascontiguousarray(w1)
        a2 = None if w2 is None else np.ascontiguousarray(w2, dtype=np.float32)
        check(lib.moe_set_predictor_mlp(self._h, layer, slot, _p(a1) if a1 is not None else None,
                                        _p(a2) if a2 is not None else None))

    def set_placement(self, layer: int, replica_counts, replica_gpu) -> None:
        rc, rg = _i32(replica_counts), _i32(replica_gpu)
        check(lib.moe_set_placement(self._h, layer, _p(rc), _p(rg)))

    # torch-tensor device entry points --------------------------------
    def gate(self, layer: int, x, ids, weights, counts, pred_counts=None, stream: int = 0) -> None:
        check(lib.moe_gate_topk(self._h, layer, x.data_ptr(), x.shape[0], ids.data_ptr(),
                                weights.data_ptr(), counts.data_ptr(),
                                pred_counts.data_ptr() if pred_counts is not None else None,
                                stream or None))

    def predict_loads(self, layer: int, x, pred_counts, stream: int = 0) -> None:
        check(lib.moe_predict_loads(self._h, layer, x.data_ptr(), x.shape[0], pred_counts.data_ptr(),
                                    stream or None))

    def forward(self, layer: int, x, y, plan_mode: int = MOE_PLAN_FIXED, iteration: int = 0,
                stats: bool = False, stream: int = 0) -> Optional[MoeLayerStats]:
        st = MoeLayerStats() if stats else None
        check(lib.moe_layer_forward(self._h, layer, x.data_ptr(), x.shape[0], y.data_ptr(), plan_mode,
                                    iteration, C.byref(st) if st is not None else None, stream or None))
        return st

    def graph_begin(self) -> None:
        """Start recording forwards into one CUDA graph (moe_graph_begin): the
        forward() calls until graph_end() are captured, not run."""
        check(lib.moe_graph_begin(self._h))

    def graph_end(self) -> int:
        """Instantiate the recorded forwards; returns the graph id."""
        gid = C.c_int(-1)
        check(lib.moe_graph_end(self._h, C.byref(gid)))
        return gid.value

    def graph_launch(self, graph_id: int, stream: int = 0) -> None:
        check(lib.moe_graph_launch(self._h, graph_id, stream or None))

    def forward_ids(self, layer: int, x, ids, y, weights=None, plan_mode: int = MOE_PLAN_FIXED,
                    iteration: int = 0, stats: bool = False, stream: int = 0) -> Optional[MoeLayerStats]:
        """The layer on caller-given routing: ids [T, k] int32 (and optional
        weights [T, k] fp32) device tensors replace the gate (K1)."""
        st = MoeLayerStats() if stats else None
        check(lib.moe_layer_forward_ids(self._h, layer, x.data_ptr(), ids.data_ptr(),
                                        weights.data_ptr() if weights is not None else None, x.shape[0],
                                        y.data_ptr(), plan_mode, iteration,
                                        C.byref(st) if st is not None else None, stream or None))
        return st

    def last_plan(self):
        """(n_e [E], segments [nseg, 3] = (first row, rows, weight slot), rows_local)
        of the dispatch plan the device used for the most recent forward."""
        n_e = np.zeros(self.E, np.int32)
        segs = np.zeros((512, 3), np.int32)
        n, rows = C.c_int(), C.c_int64()
        check(lib.moe_last_plan(self._h, _p(n_e), _p(segs), 512, C.byref(n), C.byref(rows)))
        return n_e, segs[:n.value].copy(), rows.value

    def placement(self, layer: int) -> Tuple[np.ndarray, np.ndarray]:
        """(replica_counts [E], replica_gpu [sum R]) in force for `layer`."""
        rc = np.zeros(self.E, np.int32)
        rg = np.zeros(512, np.int32)
        n = C.c_int()
        check(lib.moe_get_placement(self._h, layer, _p(rc), _p(rg), 512, C.byref(n)))
        return rc, rg[:n.value].copy()

    def forward_host(self, layer: int, x_host: np.ndarray, y_host: np.ndarray,
                     plan_mode: int = MOE_PLAN_FIXED, iteration: int = 0, stats: bool = False):
        """HOST buffers in and out (H2D + forward + D2H): the e2e call."""
        st = MoeLayerStats() if stats else None
        xp = x_host.ctypes.data if isinstance(x_host, np.ndarray) else x_host.data_ptr()
        yp = y_host.ctypes.data if isinstance(y_host, np.ndarray) else y_host.data_ptr()
        check(lib.moe_layer_forward_host(self._h, layer, C.c_void_p(xp), int(x_host.shape[0]),
                                         C.c_void_p(yp), plan_mode, iteration,
                                         C.byref(st) if st is not None else None))
        return st

    def forward_host_async(self, layer: int, x_host, y_host, plan_mode: int = MOE_PLAN_FIXED,
                           iteration: int = 0) -> int:
        """Pipelined e2e call (pinned host buffers); returns a ticket for wait()."""
        xp = x_host.ctypes.data if isinstance(x_host, np.ndarray) else x_host.data_ptr()
        yp = y_host.ctypes.data if isinstance(y_host, np.ndarray) else y_host.data_ptr()
        t = C.c_int64()
        check(lib.moe_layer_forward_host_async(self._h, layer, C.c_void_p(xp), int(x_host.shape[0]),
                                               C.c_void_p(yp), plan_mode, iteration, C.byref(t)))
        return t.value

    def gemm_times(self, max_n: int = 64):
        """(gemm1_ms, gemm2_ms, rows) of the most recent forwards (event ring, no per-step sync)."""
        g1, g2 = np.zeros(max_n, np.float32), np.zeros(max_n, np.float32)
        rows = np.zeros(max_n, np.int64)
        n = C.c_int()
        check(lib.moe_gemm_times(self._h, max_n, _p(g1), _p(g2), _p(rows), C.byref(n)))
        return g1[:n.value], g2[:n.value], rows[:n.value]

    def wait(self, ticket: int) -> None:
        check(lib.moe_wait(self._h, ticket))

    # staged forward (external exchange) ------------------------------
    def begin(self, layer: int, x, counts_all: Optional[np.ndarray] = None) -> None:
        ca = _i32(np.asarray(counts_all).reshape(-1)) if counts_all is not None else None
        check(lib.moe_forward_begin(self._h, layer, x.data_ptr(), x.shape[0],
                                    _p(ca) if ca is not None else None, None))

    def expert(self, layer: int) -> None:
        check(lib.moe_forward_expert(self._h, layer, None))

    def end(self, y) -> None:
        check(lib.moe_forward_end(self._h, y.data_ptr(), None))

    def memcpy(self, dst: int, src: int, nbytes: int) -> None:
        check(lib.moe_memcpy(self._h, C.c_void_p(dst), C.c_void_p(src), nbytes))

    def read_buffer(self, which: int, dtype, shape) -> np.ndarray:
        """Copy a ctx device buffer (see moe_buffer ids) to a new host array."""
        ptr, _ = self.buffer(which)
        out = np.empty(shape, dtype)
        if out.nbytes:
            self.memcpy(out.ctypes.data, ptr, out.nbytes)
        return out

    def buffer(self, which: int) -> Tuple[int, int]:
        p, rows = C.c_void_p(), C.c_int64()
        check(lib.moe_buffer(self._h, which, C.byref(p), C.byref(rows)))
        return p.value or 0, rows.value
