"""ctypes binding of libsparse2d_b200.so (include/sparse2d_b200.h).

The library is built in-tree by ``paper_2508_03854_b200.build``.  There is no
fallback: if the shared library is missing or cannot be loaded, importing the
device API raises, so a GPU run can never silently use another code path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = _build.LIB

S2D_OK, S2D_EINVAL, S2D_ERANGE, S2D_ENONFINITE, S2D_ERUNTIME, S2D_ECUDA, S2D_ENCCL = range(7)
S2D_TABLE_WISE, S2D_ROW_WISE = 0, 1
S2D_ROWWISE_ADAGRAD, S2D_SGD = 0, 1
S2D_F32, S2D_BF16 = 0, 1
S2D_HOST, S2D_DEVICE = 0, 1
S2D_POOL_SUM, S2D_POOL_MEAN = 0, 1


class TableLoadProfile(C.Structure):
    _fields_ = [("table_id", C.c_uint32), ("size_bytes", C.c_uint64),
                ("expected_lookups_per_batch", C.c_double), ("num_rows", C.c_uint64)]


class PlanEntry(C.Structure):
    _fields_ = [("table_id", C.c_uint32), ("row_lo", C.c_uint32), ("row_hi", C.c_uint32),
                ("local_rank", C.c_uint32)]


class OptimizerConfigC(C.Structure):
    _fields_ = [("eta", C.c_double), ("eps", C.c_double), ("c", C.c_double), ("variant", C.c_int32)]


class TopologyC(C.Structure):
    _fields_ = [("total_ranks", C.c_uint32), ("groups", C.c_uint32), ("ranks_per_group", C.c_uint32)]


class TableDesc(C.Structure):
    _fields_ = [("table_id", C.c_uint32), ("rows", C.c_uint32), ("dim", C.c_uint32), ("pooling", C.c_uint32)]


class StepStats(C.Structure):
    _fields_ = [("nnz_local", C.c_uint64), ("nnz_owned", C.c_uint64), ("entries_owned", C.c_uint64),
                ("unique_rows", C.c_uint64), ("long_segments", C.c_uint64), ("dirty_rows", C.c_uint64),
                ("a2a_bytes_sent", C.c_uint64), ("a2a_bytes_recv", C.c_uint64), ("sync_bytes", C.c_uint64),
                ("error_flags", C.c_uint32), ("sync_mode", C.c_uint32), ("ids_bytes_sent", C.c_uint64),
                ("lookup_bytes_sent", C.c_uint64), ("grad_bytes_sent", C.c_uint64), ("host_wait_ns", C.c_uint64)]


class TrainerOptionsC(C.Structure):
    _fields_ = [("total_ranks", C.c_uint32), ("groups", C.c_uint32), ("num_tables", C.c_uint32),
                ("rows_per_table", C.c_uint32), ("dim", C.c_uint32), ("strategy", C.c_int32),
                ("zipf_exponent", C.c_double), ("ids_per_sample", C.c_uint32), ("per_rank_batch", C.c_uint32),
                ("steps", C.c_uint64), ("sync_interval", C.c_uint32), ("data_seed", C.c_uint64),
                ("init_seed", C.c_uint64), ("opt", OptimizerConfigC), ("weight_dtype", C.c_int32),
                ("n_devices", C.c_uint32), ("devices", C.POINTER(C.c_int32)), ("dense_model", C.c_int32),
                ("dense_dim", C.c_uint32), ("dense_hidden", C.c_uint32), ("over_hidden", C.c_uint32),
                ("gt_id_scale", C.c_double), ("gt_dense_scale", C.c_double), ("gt_bias", C.c_double),
                ("eval_cadence", C.c_uint64), ("eval_samples", C.c_uint32), ("eval_seed", C.c_uint64)]


class TrainMetricsRowC(C.Structure):
    _fields_ = [("step", C.c_uint64), ("loss", C.c_double), ("ne", C.c_double), ("eff_lr_p50", C.c_double),
                ("eff_lr_p99", C.c_double), ("v_mean", C.c_double)]


class NEReportC(C.Structure):
    _fields_ = [("ne", C.c_double), ("baseline_ctr", C.c_double), ("eval_samples", C.c_uint64)]


UPSTREAM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p,
                          C.c_void_p, C.c_void_p)


class MetricsRowC(C.Structure):
    _fields_ = [("eff_lr_p50", C.c_double), ("eff_lr_p99", C.c_double), ("v_mean", C.c_double),
                ("rows", C.c_uint64)]


# symbol -> (restype, argtypes); the full exported surface of the header
_P = C.c_void_p
SIGNATURES = {
    "s2d_last_error": (C.c_char_p, []),
    "s2d_version": (C.c_char_p, []),
    "s2d_topology_init": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(TopologyC)]),
    "s2d_plan_greedy": (C.c_int, [C.POINTER(TableLoadProfile), C.c_uint32, C.c_uint32, C.c_int32,
                                  C.POINTER(PlanEntry), C.c_uint32, C.POINTER(C.c_uint32)]),
    "s2d_validate_plan": (C.c_int, [C.POINTER(PlanEntry), C.c_uint32, C.c_uint32,
                                    C.POINTER(TableLoadProfile), C.c_uint32]),
    "s2d_plan_owner_of": (C.c_int, [C.POINTER(PlanEntry), C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_uint32)]),
    "s2d_imbalance_ratio": (C.c_int, [C.POINTER(C.c_double), C.c_uint32, C.POINTER(C.c_double)]),
    "s2d_effective_lr": (C.c_int, [C.c_double, C.POINTER(OptimizerConfigC), C.POINTER(C.c_double)]),
    "s2d_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "s2d_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "s2d_ctx_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_char_p, C.POINTER(_P)]),
    "s2d_ctx_destroy": (C.c_int, [_P]),
    "s2d_hub_create": (C.c_int, [C.c_uint32, C.POINTER(_P)]),
    "s2d_hub_destroy": (C.c_int, [_P]),
    "s2d_ctx_create_local": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, _P, C.POINTER(_P)]),
    "s2d_ctx_set_stream": (C.c_int, [_P, _P]),
    "s2d_ctx_set_strict": (C.c_int, [_P, C.c_int]),
    "s2d_ctx_set_async_host": (C.c_int, [_P, C.c_int]),
    "s2d_save_tables": (C.c_int, [_P, C.c_char_p]),
    "s2d_load_tables": (C.c_int, [_P, C.c_char_p]),
    "s2d_gen_batch": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, _P, _P, _P, _P, C.c_int32]),
    "s2d_register_tables": (C.c_int, [_P, C.POINTER(TableDesc), C.c_uint32, C.POINTER(PlanEntry), C.c_uint32,
                                      C.c_int32]),
    "s2d_set_optimizer": (C.c_int, [_P, C.POINTER(OptimizerConfigC)]),
    "s2d_init_tables": (C.c_int, [_P, C.c_uint64]),
    "s2d_shard_write": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, _P, _P]),
    "s2d_apply_row_updates": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P]),
    "s2d_shard_read": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, _P, _P]),
    "s2d_shard_range": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "s2d_lookup_forward": (C.c_int, [_P, C.c_uint32, _P, _P, C.c_uint64, _P, C.c_int32]),
    "s2d_backward_update": (C.c_int, [_P, _P, C.c_int32]),
    "s2d_pooled_buffer": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "s2d_replica_sync": (C.c_int, [_P]),
    "s2d_synchronize": (C.c_int, [_P]),
    "s2d_get_step_stats": (C.c_int, [_P, C.POINTER(StepStats)]),
    "s2d_adagrad_rows": (C.c_int, [C.POINTER(OptimizerConfigC), C.c_uint32, C.c_uint32, _P, _P, _P, _P]),
    "s2d_ctx_set_profiling": (C.c_int, [_P, C.c_int]),
    "s2d_get_phase_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.c_uint32]),
    "s2d_launch_count": (C.c_uint64, []),
    "s2d_metrics": (C.c_int, [_P, C.POINTER(MetricsRowC)]),
    "s2d_shard_gather": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P]),
    "s2d_ctx_set_debug_grad": (C.c_int, [_P, C.c_int]),
    "s2d_gen_upstream": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, _P, C.c_int32]),
    "s2d_trainer_create": (C.c_int, [C.POINTER(TrainerOptionsC), C.POINTER(_P)]),
    "s2d_trainer_destroy": (C.c_int, [_P]),
    "s2d_trainer_set_upstream": (C.c_int, [_P, UPSTREAM_FN, _P]),
    "s2d_trainer_step_n": (C.c_int, [_P, C.c_uint64]),
    "s2d_trainer_run": (C.c_int, [_P]),
    "s2d_trainer_steps_done": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "s2d_trainer_plan": (C.c_int, [_P, C.POINTER(PlanEntry), C.c_uint32, C.POINTER(C.c_uint32)]),
    "s2d_trainer_replica_table": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P]),
    "s2d_trainer_save_tables": (C.c_int, [_P, C.c_char_p]),
    "s2d_trainer_load_tables": (C.c_int, [_P, C.c_char_p]),
    "s2d_trainer_metrics": (C.c_int, [_P, C.POINTER(MetricsRowC)]),
    "s2d_trainer_rank_ctx": (C.c_int, [_P, C.c_uint32, C.POINTER(_P)]),
    "s2d_trainer_rank_model": (C.c_int, [_P, C.c_uint32, C.c_int32, _P, _P, _P, _P]),
    "s2d_trainer_last_loss": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "s2d_pool_ids": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _P, _P, C.c_uint64, _P, _P, _P]),
    "s2d_aggregate_group_gradient": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, C.c_uint32, _P, _P, _P, C.c_uint64,
                                               C.POINTER(C.c_uint64)]),
    "s2d_trainer_metrics_rows": (C.c_int, [_P, _P, C.c_uint32, C.POINTER(C.c_uint32)]),
    "s2d_trainer_final_ne": (C.c_int, [_P, C.POINTER(NEReportC)]),
    "s2d_memory_overhead": (C.c_int, [C.c_double, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]),
    "s2d_sync_latency": (C.c_int, [C.c_double, C.c_uint32, C.c_uint32, C.c_double, C.POINTER(C.c_double)]),
    "s2d_qps_scaling_factor": (C.c_int, [C.c_double] * 4 + [C.POINTER(C.c_double)]),
    "s2d_evaluate_ne": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "s2d_closed_form_ratio": (C.c_int, [C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.POINTER(C.c_double)]),
    "s2d_recommend_c": (C.c_int, [C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]),
    "s2d_estimate_increment_ratio": (C.c_int, [C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint64, C.c_uint64, C.POINTER(C.c_double),
                                               C.POINTER(C.c_double)]),
    "s2d_debug_read": (C.c_int, [_P, C.c_int32, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
}

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed and nvcc is available) the library.
    Raises if it cannot be loaded -- there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    # SPARSE2D_EXT_DIR (python/sparse2d/__init__.py:8-10): a prebuilt library
    # in that directory is used as is
    ext = os.environ.get("SPARSE2D_EXT_DIR")
    if ext and os.path.exists(os.path.join(ext, os.path.basename(LIB_PATH))):
        _lib = _bind(C.CDLL(os.path.join(ext, os.path.basename(LIB_PATH))))
        return _lib
    if not _build.up_to_date():
        if not build_if_missing:
            raise ImportError(f"{LIB_PATH} missing or stale; run python -m paper_2508_03854_b200.build")
        _build.build()
    _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def _bind(lib: C.CDLL) -> C.CDLL:
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class Sparse2DError(RuntimeError):
    pass


_EXC = {
    S2D_EINVAL: ValueError,       # std::invalid_argument (pybind -> ValueError)
    S2D_ERANGE: IndexError,       # std::out_of_range -> IndexError
    S2D_ENONFINITE: ValueError,   # invalid_argument("nonfinite row gradient")
    S2D_ERUNTIME: RuntimeError,
    S2D_ECUDA: Sparse2DError,
    S2D_ENCCL: Sparse2DError,
}


def check(rc: int) -> None:
    if rc != S2D_OK:
        msg = _lib.s2d_last_error().decode() if _lib is not None else "error"
        raise _EXC.get(rc, RuntimeError)(msg)
