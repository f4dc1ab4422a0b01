"""ctypes binding of ``libautoshard_b200.so`` (include/autoshard_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2208_06399_b200/csrc``). There is no fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AUTOSHARD_B200_LIB") or os.path.join(HERE, "libautoshard_b200.so")


class TableSpecC(C.Structure):
    _fields_ = [
        ("id", C.c_int32),
        ("dim", C.c_int32),
        ("hash_size", C.c_int64),
        ("pooling_mean", C.c_double),
        ("access_ratio", C.c_double),
        ("bytes_per_param", C.c_int32),
        ("_pad", C.c_int32),
    ]


class GeneratorConfigC(C.Structure):
    _fields_ = [
        ("hash_size_min", C.c_double),
        ("hash_size_max", C.c_double),
        ("pooling_mean_target", C.c_double),
        ("pooling_shape", C.c_double),
        ("pooling_cap", C.c_double),
        ("dim_choices", C.POINTER(C.c_int32)),
        ("n_dim_choices", C.c_int32),
        ("access_ratio_min", C.c_double),
        ("access_ratio_max", C.c_double),
        ("bytes_per_param", C.c_int32),
    ]


class BenchConfigC(C.Structure):
    _fields_ = [
        ("warmup", C.c_int32),
        ("measure", C.c_int32),
        ("trim", C.c_int32),
        ("flush_l2", C.c_int32),
        ("seed", C.c_uint64),
        ("lr", C.c_float),
        ("eps", C.c_float),
    ]


class CtxInfoC(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("n_tables", C.c_int32),
        ("batch_size", C.c_int64),
        ("sum_dim", C.c_int64),
        ("total_rows", C.c_int64),
        ("n_lookups", C.c_int64),
        ("n_chunks", C.c_int64),
        ("device_bytes", C.c_int64),
        ("pooled", C.c_void_p),
        ("weights", C.c_void_p),
        ("momentum", C.c_void_p),
        ("kernels_per_step", C.c_int32),
        ("weight_bytes", C.c_int32),
    ]


class CommInfoC(C.Structure):
    """as_comm_info."""

    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("mode", C.c_int32),
        ("has_nccl", C.c_int32),
        ("recv_rows", C.c_int64),
        ("recv_cols", C.c_int64),
        ("recv", C.c_void_p),
        ("grad", C.c_void_p),
        ("bytes_sent_fwd", C.c_int64),
        ("bytes_sent_bwd", C.c_int64),
    ]


P = C.POINTER
i32, i64, u64, f32, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p
T_SPEC = P(TableSpecC)

# name -> (restype, argtypes); every symbol declared in include/autoshard_b200.h
SIGNATURES = {
    "as_version": (C.c_char_p, []),
    "as_last_error": (C.c_char_p, []),
    "as_generator_config_default": (None, [P(GeneratorConfigC)]),
    "as_generate_pool": (i32, [u64, i32, P(GeneratorConfigC), T_SPEC]),
    "as_generate_workload": (i32, [u64, T_SPEC, i32, i64, f64, i32, P(vp)]),
    "as_workload_batch_size": (i64, [vp]),
    "as_workload_num_tables": (i32, [vp]),
    "as_workload_stream": (i32, [vp, i32, P(i32), P(P(i64)), P(P(i64)), P(i64)]),
    "as_workload_find": (i32, [vp, i32, P(i32)]),
    "as_workload_from_arrays": (i32, [i64, i32, P(i32), P(vp), P(vp), P(i64), P(vp)]),
    "as_workload_pin": (i32, [vp]),
    "as_workload_destroy": (None, [vp]),
    "as_workload_save": (i32, [vp, T_SPEC, C.c_char_p]),
    "as_workload_load": (i32, [C.c_char_p, P(vp), T_SPEC, i32, P(i32)]),
    "as_pool_save": (i32, [T_SPEC, i32, C.c_char_p]),
    "as_pool_load": (i32, [C.c_char_p, T_SPEC, i32, P(i32)]),
    "as_fingerprint_pool": (u64, [T_SPEC, i32]),
    "as_fingerprint_task": (u64, [T_SPEC, i32, i32, P(i64)]),
    "as_heuristic_cost": (i32, [T_SPEC, i32, P(f64)]),
    "as_greedy_shard": (i32, [T_SPEC, i32, i32, P(i64), i32, P(i32)]),
    "as_random_shard": (i32, [T_SPEC, i32, i32, P(i64), u64, P(i32)]),
    "as_plan_validate": (i32, [i32, i32, P(i32)]),
    "as_plan_mem_used": (i32, [T_SPEC, i32, i32, P(i32), P(i64)]),
    "as_degree_of_balance": (i32, [P(f64), i32, P(f64)]),
    "as_plan_save": (i32, [C.c_char_p, T_SPEC, i32, i32, P(i64), P(i32), P(f64)]),
    "as_plan_load": (i32, [C.c_char_p, T_SPEC, i32, i32, P(i64), P(i32), P(f64), P(i32)]),
    "as_create": (i32, [i32, T_SPEC, i32, i64, u64, P(vp)]),
    "as_create_ex": (i32, [i32, T_SPEC, i32, i64, u64, i32, P(vp)]),
    "as_destroy": (i32, [vp]),
    "as_create_subset": (i32, [vp, P(i32), i32, P(vp)]),
    "as_retarget_subset": (i32, [vp, P(i32), i32]),
    "as_load_streams_exchanged": (i32, [vp, i32, T_SPEC, P(i32), P(vp), P(vp), vp]),
    "as_load_streams": (i32, [vp, P(vp), P(vp), P(i64), vp]),
    "as_load_workload": (i32, [vp, vp, vp]),
    "as_stage_streams": (i32, [vp, P(vp), P(vp), P(i64)]),
    "as_stage_workload": (i32, [vp, vp]),
    "as_commit_staged": (i32, [vp, vp]),
    "as_check_batch": (i32, [vp]),
    "as_forward": (i32, [vp, vp, vp]),
    "as_set_peer_outputs": (i32, [vp, i32, P(vp), i64]),
    "as_backward_rowwise_adagrad": (i32, [vp, vp, f32, f32, vp]),
    "as_step": (i32, [vp, f32, f32, P(f64), vp]),
    "as_measure": (i32, [vp, i32, i32, i32, i32, f32, f32, P(f64)]),
    "as_measure_plan": (i32, [T_SPEC, i32, i32, P(i32), vp, P(i32), i32, P(BenchConfigC), P(f64)]),
    "as_ctx_info_get": (i32, [vp, P(CtxInfoC)]),
    "as_profile_enable": (i32, [vp, i32]),
    "as_profile_read": (i32, [vp, P(f64), P(i64), i32]),
    "as_table_features": (i32, [vp, P(f64), vp]),
    "as_probe_gather_bw": (i32, [i32, i64, i32, P(f64)]),
    "as_set_peer_outputs_v": (i32, [vp, i32, P(vp), P(i64)]),
    "as_comm_unique_id": (i32, [vp]),
    "as_comm_init": (i32, [vp, vp, i32, i32, P(vp)]),
    "as_comm_destroy": (i32, [vp]),
    "as_alltoall_setup": (i32, [vp, P(i64), P(i64), i32]),
    "as_alltoall_handle": (i32, [vp, vp, P(i64)]),
    "as_alltoall_open": (i32, [vp, vp]),
    "as_alltoall_host_barrier": (i32, [vp, vp, vp]),
    "as_forward_sharded": (i32, [vp, vp]),
    "as_backward_sharded": (i32, [vp, vp, f32, f32, vp]),
    "as_step_sharded": (i32, [vp, f32, f32, P(f64), vp]),
    "as_comm_info_get": (i32, [vp, P(CommInfoC)]),
    "as_comm_profile_read": (i32, [vp, P(f64), i32]),
    "as_read_rows": (i32, [vp, i32, P(i64), i64, P(f32)]),
    "as_read_momentum": (i32, [vp, i32, P(i64), i64, P(f32)]),
    "as_read_buffer": (i32, [vp, i32, vp, i64]),
    "as_write_table": (i32, [vp, i32, P(f32), P(f32)]),
}

_lib = None


def lib():
    """Load the C-ABI library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
