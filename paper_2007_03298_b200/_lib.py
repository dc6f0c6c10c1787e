"""ctypes binding of the C-ABI in include/dssync_b200.h.

Loads the in-tree ``libdssync_b200.so``.  There is no fallback: if the
library is missing the import fails loudly (the product path is the CUDA
library or nothing).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdssync_b200.so")
# Tuning experiments only: load a variant build of the same library
# (paper_2007_03298_b200.build --variant); the product default is LIB_PATH.
LIB_PATH = os.environ.get("DSS_LIB_VARIANT", LIB_PATH)

DSS_OK, DSS_EINVAL, DSS_EDIVERGED, DSS_ECUDA, DSS_ENCCL, DSS_ERUNTIME = range(6)
DSS_F32, DSS_F64 = 0, 1
BUF_PARAMS, BUF_GRADS, BUF_MOMENT1, BUF_MOMENT2, BUF_STATS, BUF_STATS_OBS = range(6)
SAMPLING_REPLACEMENT, SAMPLING_EPOCH = 0, 1  # dss_sampling
IPC_BYTES = 736
KIND_NAMES = ["group", "fold", "bsp", "barrier", "gradient", "chain", "chain_mean"]


class dss_hparams(C.Structure):
    _fields_ = [("momentum", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("epsilon", C.c_double), ("weight_decay", C.c_double)]


class dss_strategy(C.Structure):
    _fields_ = [("kind", C.c_int), ("topology", C.c_int), ("world_size", C.c_int),
                ("group_size", C.c_int), ("num_servers", C.c_int), ("rectangular", C.c_int)]


class dss_outcome(C.Structure):
    _fields_ = [("critical_path_steps", C.c_long), ("total_messages", C.c_long)]


class dss_config(C.Structure):
    _fields_ = [("strategy", dss_strategy), ("optimizer", C.c_int), ("hp", dss_hparams),
                ("dtype", C.c_int), ("dim", C.c_long), ("device", C.c_int), ("rank", C.c_int),
                ("n_gpus", C.c_int), ("path", C.c_int), ("stats_dim", C.c_long), ("placement", C.c_int)]


class dss_plan_summary(C.Structure):
    _fields_ = [("local_groups", C.c_int), ("spanning_groups", C.c_int),
                ("owned_slices", C.c_int), ("owned_elems", C.c_long), ("chain_groups", C.c_int)]


# Every symbol declared in include/dssync_b200.h, with its signature.
_P = C.c_void_p
SIGNATURES = {
    "dss_validate_world": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "dss_validate_strategy": (C.c_int, [C.POINTER(dss_strategy)]),
    "dss_is_square_mode": (C.c_int, [C.c_int, C.c_int]),
    "dss_partition": (C.c_int, [C.POINTER(dss_strategy), C.c_long, _P, _P, C.POINTER(C.c_int)]),
    "dss_group_of": (C.c_int, [C.POINTER(dss_strategy), C.c_long, C.c_int, _P, C.POINTER(C.c_int)]),
    "dss_check_mixing": (C.c_int, [C.POINTER(dss_strategy), C.c_long]),
    "dss_round_outcome": (C.c_int, [C.POINTER(dss_strategy), C.c_long, C.c_long, C.POINTER(dss_outcome)]),
    "dss_plan": (C.c_int, [C.POINTER(dss_strategy), C.c_long, C.c_long, C.c_int, C.c_int,
                           C.POINTER(dss_plan_summary), _P, _P, _P, C.c_int]),
    "dss_create": (C.c_int, [C.POINTER(dss_config), C.POINTER(_P)]),
    "dss_destroy": (C.c_int, [_P]),
    "dss_set_stream": (C.c_int, [_P, _P]),
    "dss_local_workers": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "dss_local_ranks": (C.c_int, [_P, _P]),
    "dss_placement": (C.c_int, [C.POINTER(dss_strategy), C.c_int, C.c_int, C.c_long, C.c_int, _P, _P,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "dss_row_stride": (C.c_long, [_P]),
    "dss_elem_size": (C.c_int, [_P]),
    "dss_device_ptr": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(_P)]),
    "dss_upload": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_long]),
    "dss_download": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_long]),
    "dss_upload_all": (C.c_int, [_P, C.c_int, _P]),
    "dss_download_all": (C.c_int, [_P, C.c_int, _P]),
    "dss_broadcast_row": (C.c_int, [_P, C.c_int, _P]),
    "dss_set_step_count": (C.c_int, [_P, C.c_int, C.c_long]),
    "dss_get_step_count": (C.c_long, [_P, C.c_int]),
    "dss_step": (C.c_int, [_P, C.c_long, C.c_double, C.c_int, C.POINTER(dss_outcome)]),
    "dss_steps": (C.c_int, [_P, C.c_long, C.c_long, _P, C.c_int, C.POINTER(dss_outcome)]),
    "dss_step_host": (C.c_int, [_P, C.c_long, C.c_double, _P, _P]),
    "dss_host_sync": (C.c_int, [_P]),
    "dss_sync_round": (C.c_int, [_P, C.c_long, C.c_int, C.POINTER(dss_outcome)]),
    "dss_apply_step": (C.c_int, [_P, C.c_double, C.c_int]),
    "dss_running_stats_update": (C.c_int, [_P]),
    "dss_quadratic_gradients": (C.c_int, [_P, C.c_long, C.c_uint64, C.c_double, C.c_double]),
    "dss_quadratic_init": (C.c_int, [_P, C.c_uint64, C.c_double]),
    "dss_set_optimum": (C.c_int, [_P, _P, C.c_long]),
    "dss_global_mean": (C.c_int, [_P, _P]),
    "dss_quadratic_losses": (C.c_int, [_P, C.c_double, C.c_int, _P, _P]),
    "dss_logistic_dataset": (C.c_int, [C.c_uint64, C.c_int, C.c_int, _P, _P]),
    "dss_quadratic_problem": (C.c_int, [C.c_uint64, C.c_int, C.c_double, _P, _P]),
    "dss_logistic_constants": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_double, _P, _P, _P]),
    "dss_mlp_dataset": (C.c_int, [C.c_uint64, C.c_int, C.c_int, _P, _P]),
    "dss_mlp_initial_params": (C.c_int, [C.c_uint64, C.c_int, C.c_int, _P]),
    "dss_mlp_setup": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64]),
    "dss_mlp_gradients": (C.c_int, [_P, C.c_long]),
    "dss_mlp_losses": (C.c_int, [_P, C.c_int, _P]),
    "dss_make_shards": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _P, _P]),
    "dss_epoch_order": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_int, C.c_long, _P]),
    "dss_logistic_setup": (C.c_int, [_P, _P, _P, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64]),
    "dss_logistic_gradients": (C.c_int, [_P, C.c_long]),
    "dss_logistic_steps": (C.c_int, [_P, C.c_long, C.c_long, _P, C.c_int, _P]),
    "dss_logistic_batch": (C.c_int, [_P, _P]),
    "dss_logistic_losses": (C.c_int, [_P, C.c_int, _P]),
    "dss_check": (C.c_int, [_P]),
    "dss_clear_error": (C.c_int, [_P]),
    "dss_last_error": (C.c_int, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_long)]),
    "dss_last_global_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "dss_enable_timing": (C.c_int, [_P, C.c_int]),
    "dss_kernel_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_long), C.POINTER(C.c_double)]),
    "dss_kernel_times_by_kind": (C.c_int, [_P, _P, _P]),
    "dss_launch_count": (C.c_long, [_P]),
    "dss_ipc_export": (C.c_int, [_P, _P]),
    "dss_ipc_attach": (C.c_int, [_P, _P]),
    "dss_barrier": (C.c_int, [_P]),
    "dss_check_guards": (C.c_int, [_P, C.POINTER(C.c_long)]),
    "dss_emulate_attach": (C.c_int, [_P, C.c_int]),
    "dss_emulate_step": (C.c_int, [_P, C.c_int, C.c_long, C.c_double, C.c_int]),
}

_lib = None


def load() -> C.CDLL:
    """Load the CUDA C-ABI library; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2007_03298_b200.build` "
                "(there is no CPU fallback for the DS-Sync path)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def global_error() -> str:
    buf = C.create_string_buffer(1024)
    load().dss_last_global_error(buf, len(buf))
    return buf.value.decode()
