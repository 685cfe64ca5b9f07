"""ctypes binding of the C-ABI in include/moe_b200.h (libmoe_b200.so).

The product library is loaded from the package directory (built in-tree by
`make -C paper_2603_06350_b200/csrc`).  There is no fallback: if the shared
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoe_b200.so")

MOE_OK, MOE_EINVAL, MOE_EINFEASIBLE, MOE_ECUDA, MOE_ENCCL, MOE_ESTATE = range(6)
MOE_EXCHANGE_NCCL, MOE_EXCHANGE_EXTERNAL, MOE_EXCHANGE_P2P, MOE_EXCHANGE_COPY = 0, 1, 2, 3
MOE_PLAN_FIXED, MOE_PLAN_SYNC, MOE_PLAN_PREDICTED = 0, 1, 2
MOE_PRECISION_BF16, MOE_PRECISION_FP32 = 0, 1
MOE_RESIDENCY_ALL, MOE_RESIDENCY_PLACED = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
        "(there is no CPU fallback for the MoE data path)")

lib = C.CDLL(LIB_PATH)

i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


class MoeCtxDesc(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int), ("num_experts", C.c_int), ("top_k", C.c_int),
        ("d_model", C.c_int), ("d_ff", C.c_int), ("max_tokens", C.c_int),
        ("world_size", C.c_int), ("rank", C.c_int), ("device", C.c_int),
        ("exchange_mode", C.c_int), ("nccl_unique_id", vp),
        ("num_predictor_targets", C.c_int),
        ("expert_mem_mb", dbl), ("layer_mem_cap_mb", dbl), ("gpu_mem_capacity_mb", dbl),
        ("cv_threshold", dbl), ("keep_alive_iters", C.c_int), ("predictor_distance", C.c_int),
        ("precision", C.c_int), ("use_cuda_graphs", C.c_int), ("residency", C.c_int),
        ("replica_slots", C.c_int), ("reserved", C.c_int * 2),
    ]


class MoeLayerStats(C.Structure):
    _fields_ = [
        ("compute_ms", dbl), ("comm_ms", dbl), ("forward_ms", dbl), ("replica_count", C.c_int),
        ("mem_mb", dbl), ("gate_ms", dbl), ("plan_ms", dbl), ("dispatch_ms", dbl),
        ("a2a_dispatch_ms", dbl), ("gemm1_ms", dbl), ("gemm2_ms", dbl),
        ("a2a_combine_ms", dbl), ("combine_ms", dbl), ("rows_local", i64), ("rows_sent", i64),
        ("warm_count", C.c_int), ("cold_count", C.c_int), ("counts", i32 * 256),
        ("predictor_accuracy", dbl), ("plan_source", i32),
        ("weight_copies", i32), ("weight_hits", i32), ("weight_copy_ms", dbl), ("weight_copy_mb", dbl),
    ]


class MoeP2PHandle(C.Structure):
    _fields_ = [
        ("ipc", C.c_ubyte * 64), ("pid", u64), ("base", u64), ("bytes", u64),
        ("off_flags", u64), ("off_counts", u64), ("off_xp", u64), ("off_yp", u64),
        ("device", i32), ("rank", i32), ("world_size", i32), ("version", i32),
        ("off_weights", u64), ("weight_bytes", u64), ("reserved", C.c_ubyte * 40),
    ]


assert C.sizeof(MoeP2PHandle) == 192


class MoeChunk(C.Structure):
    _fields_ = [("peer", i32), ("replica", i32), ("row_offset", i64), ("rows", i64)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("moe_last_error", C.c_char_p)
_sig("moe_version", C.c_char_p)
_sig("moe_nccl_unique_id", C.c_int, vp)
_sig("moe_ctx_create", C.c_int, P(MoeCtxDesc), P(vp))
_sig("moe_ctx_destroy", C.c_int, vp)
_sig("moe_ctx_stream", C.c_int, vp, P(vp))
_sig("moe_ctx_sync", C.c_int, vp)
_sig("moe_p2p_export", C.c_int, vp, P(MoeP2PHandle))
_sig("moe_p2p_import", C.c_int, vp, P(MoeP2PHandle), C.c_int)
_sig("moe_load_expert_weights", C.c_int, vp, C.c_int, C.c_int, vp, vp, vp)
_sig("moe_set_gate_weights", C.c_int, vp, C.c_int, vp)
_sig("moe_load_expert_weights_f32", C.c_int, vp, C.c_int, C.c_int, vp, vp, vp)
_sig("moe_set_gate_weights_f32", C.c_int, vp, C.c_int, vp)
_sig("moe_set_gate_weights_device", C.c_int, vp, C.c_int, vp, vp)
_sig("moe_set_predictor_weights", C.c_int, vp, C.c_int, C.c_int, vp)
_sig("moe_set_predictor_mlp", C.c_int, vp, C.c_int, C.c_int, vp, vp)
_sig("moe_set_placement", C.c_int, vp, C.c_int, vp, vp)
_sig("moe_gate_topk", C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp)
_sig("moe_predict_loads", C.c_int, vp, C.c_int, vp, C.c_int, vp, vp)
_sig("moe_layer_forward", C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_long, P(MoeLayerStats), vp)
_sig("moe_graph_begin", C.c_int, vp)
_sig("moe_graph_end", C.c_int, vp, P(C.c_int))
_sig("moe_graph_launch", C.c_int, vp, C.c_int, vp)
_sig("moe_layer_forward_ids", C.c_int, vp, C.c_int, vp, vp, vp, C.c_int, vp, C.c_int, C.c_long, P(MoeLayerStats),
     vp)
_sig("moe_last_plan", C.c_int, vp, vp, vp, C.c_int, P(C.c_int), P(i64))
_sig("moe_get_placement", C.c_int, vp, C.c_int, vp, vp, C.c_int, P(C.c_int))
_sig("moe_layer_forward_host", C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_long, P(MoeLayerStats))
_sig("moe_layer_forward_host_async", C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_long, P(i64))
_sig("moe_wait", C.c_int, vp, i64)
_sig("moe_host_alloc", C.c_int, C.c_size_t, P(vp))
_sig("moe_gemm_times", C.c_int, vp, C.c_int, vp, vp, vp, P(C.c_int))
_sig("moe_residency", C.c_int, vp, C.c_int, vp, P(C.c_int))
_sig("moe_host_free", C.c_int, vp)
_sig("moe_forward_begin", C.c_int, vp, C.c_int, vp, C.c_int, vp, vp)
_sig("moe_forward_expert", C.c_int, vp, C.c_int, vp)
_sig("moe_forward_end", C.c_int, vp, vp, vp)
_sig("moe_buffer", C.c_int, vp, C.c_int, P(vp), P(i64))
_sig("moe_memcpy", C.c_int, vp, vp, vp, C.c_size_t)
_sig("moe_exchange_plan_direct", C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, P(i64), P(i64))
_sig("moe_exchange_plan", C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp,
     P(MoeChunk), P(C.c_int), P(MoeChunk), P(C.c_int), C.c_int, P(i64), P(i64), vp, vp)
_sig("moe_plan_scale", C.c_int, vp, C.c_int, C.c_int, dbl, dbl, dbl, C.c_int, vp, P(dbl), P(C.c_int),
     vp, vp, C.c_int)
_sig("moe_registry_create", C.c_int, C.c_int, P(vp))
_sig("moe_registry_destroy", C.c_int, vp)
_sig("moe_registry_size", i64, vp)
_sig("moe_plan_place", C.c_int, vp, vp, vp, C.c_int, C.c_int, dbl, C.c_int, dbl, C.c_long, C.c_int,
     dbl, dbl, vp, P(C.c_int), P(C.c_int))
_sig("moe_registry_update", C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_long)
_sig("moe_model_forward_time", C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp)
_sig("moe_plan_predict", C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
     dbl, C.c_int, C.c_long, u64, vp, vp, P(C.c_int))
_sig("moe_measure_accuracy", dbl, vp, vp, C.c_int)
_sig("moe_percentile", dbl, vp, C.c_int, dbl)
_sig("moe_route_tokens", C.c_int, i64, C.c_int, C.c_long, C.c_int, C.c_int, dbl, u64, C.c_int, C.c_int, vp)
_sig("moe_popularity", C.c_int, C.c_int, C.c_int, dbl, u64, C.c_int, C.c_long, C.c_int, vp, vp)
_sig("moe_static_plan", C.c_int, vp, C.c_int, C.c_int, dbl, dbl, vp)
_sig("moe_round_robin_placement", C.c_int, vp, C.c_int, C.c_int, dbl, dbl, vp)
_sig("moe_gpu_comm_times", C.c_int, vp, vp, vp, C.c_int, C.c_int, dbl, vp)
_sig("moe_oracle_balance_time", C.c_int, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp)
_sig("moe_verify_plan", C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, C.c_int, dbl, dbl, dbl, dbl, C.c_int,
     P(C.c_int), C.c_char_p, C.c_int)
_sig("moe_apply_finetuning", C.c_int, vp, C.c_int, dbl, vp)
_sig("moe_coefficient_of_variation", dbl, vp, C.c_int)
_sig("moe_serverful_cost", dbl, dbl, C.c_int, C.c_int, dbl, dbl)
_sig("moe_stream_key", u64, u64, u64, u64, u64)
_sig("moe_synth_tokens", C.c_int, u64, i64, i64, C.c_int, C.c_int, vp)
_sig("moe_synth_gate", C.c_int, u64, C.c_int, C.c_int, vp, vp, vp)
_sig("moe_synth_expert", C.c_int, u64, C.c_int, C.c_int, vp, vp, vp)

# Every symbol include/moe_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "moe_last_error", "moe_version", "moe_nccl_unique_id", "moe_ctx_create", "moe_ctx_destroy", "moe_ctx_stream",
    "moe_ctx_sync", "moe_p2p_export", "moe_p2p_import", "moe_load_expert_weights", "moe_set_gate_weights",
    "moe_load_expert_weights_f32", "moe_set_gate_weights_f32", "moe_set_gate_weights_device",
    "moe_set_predictor_weights", "moe_set_predictor_mlp", "moe_set_placement", "moe_gate_topk", "moe_predict_loads",
    "moe_layer_forward", "moe_graph_begin", "moe_graph_end", "moe_graph_launch", "moe_layer_forward_ids", "moe_last_plan", "moe_get_placement", "moe_layer_forward_host", "moe_layer_forward_host_async", "moe_wait",
    "moe_host_alloc", "moe_host_free", "moe_gemm_times", "moe_residency",
    "moe_forward_begin", "moe_forward_expert",
    "moe_forward_end", "moe_buffer", "moe_memcpy", "moe_exchange_plan", "moe_exchange_plan_direct", "moe_plan_scale",
    "moe_registry_create", "moe_registry_destroy", "moe_registry_size", "moe_plan_place",
    "moe_registry_update", "moe_model_forward_time", "moe_plan_predict", "moe_measure_accuracy",
    "moe_percentile", "moe_static_plan", "moe_round_robin_placement", "moe_gpu_comm_times",
    "moe_oracle_balance_time", "moe_verify_plan", "moe_apply_finetuning", "moe_coefficient_of_variation",
    "moe_serverful_cost", "moe_route_tokens", "moe_popularity", "moe_stream_key", "moe_synth_tokens",
    "moe_synth_gate", "moe_synth_expert",
]


class MoeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int) -> None:
    """Map a status code to the exception class the C++ shim would throw."""
    if rc == MOE_OK:
        return
    msg = (lib.moe_last_error() or b"").decode()
    if rc == MOE_EINVAL:
        raise ValueError(msg)
    raise MoeError(rc, msg)
