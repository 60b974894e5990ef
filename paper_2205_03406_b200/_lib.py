"""ctypes binding of libhpeel_b200.so (the C ABI in include/hpeel_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2205_03406_b200/csrc``). There is no fallback: if the library
is missing every call raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhpeel_b200.so")

HP_OK, HP_ERR_INVALID_ARGUMENT, HP_ERR_RUNTIME, HP_ERR_LOGIC = 0, 1, 2, 3

_lib = None

i64 = C.c_int64
u64 = C.c_uint64
P = C.c_void_p
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
lp = C.POINTER(C.c_int64)

_SIGNATURES = {
    "hp_last_error": (C.c_char_p, []),
    "hp_device_count": (C.c_int, [ip]),
    "hp_launch_count": (i64, []),
    "hp_device_synchronize": (C.c_int, []),
    "hp_mix_seed": (u64, [u64, u64]),
    "hp_gaussian_matrix": (C.c_int, [i64, i64, u64, dp]),
    "hp_random_cloud": (C.c_int, [i64, C.c_int, u64, dp]),
    "hp_tree_build": (C.c_int, [dp, i64, C.c_int, C.c_int, C.POINTER(P)]),
    "hp_tree_free": (None, [P]),
    "hp_tree_info": (C.c_int, [P, lp]),
    "hp_tree_boxes": (C.c_int, [P, ip, ip, lp, lp, ip]),
    "hp_tree_lists": (C.c_int, [P, C.c_int, lp, ip]),
    "hp_tree_cross_level_adjacencies": (i64, [P]),
    "hp_tree_pairs": (C.c_int, [P, C.c_int, lp, ip]),
    "hp_tree_layout": (C.c_int, [P, ip, lp, lp]),
    "hp_plan_build": (C.c_int, [P, C.c_int, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.POINTER(P)]),
    "hp_plan_free": (None, [P]),
    "hp_plan_info": (C.c_int, [P, lp]),
    "hp_plan_sets": (C.c_int, [P, lp, ip, ip, lp, ip, lp, ip]),
    "hp_plan_graph": (C.c_int, [P, lp, ip]),
    "hp_plan_coloring": (C.c_int, [P, ip, ip, ip]),
    "hp_plan_matrices": (C.c_int, [P, lp, ip]),
    "hp_plan_block_map": (C.c_int, [P, C.POINTER(C.c_int64), ip]),
    "hp_plan_realize": (C.c_int, [P, C.c_int, dp]),
    "hp_dsatur": (C.c_int, [C.c_int, lp, ip, ip, ip, lp]),
    "hp_op_dense": (C.c_int, [dp, i64, C.c_int, C.POINTER(P)]),
    "hp_op_kernel": (C.c_int, [C.c_int, dp, i64, C.c_int, C.c_double, C.c_int, C.POINTER(P)]),
    "hp_op_callback": (C.c_int, [i64, C.c_int, C.c_int, P, P, C.c_int, C.POINTER(P)]),
    "hp_op_free": (None, [P]),
    "hp_op_apply": (C.c_int, [P, C.c_int, dp, i64, dp]),
    "hp_compress": (C.c_int, [P, P, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "hp_rep_free": (None, [P]),
    "hp_comm_unique_id": (C.c_int, [C.c_char_p]),
    "hp_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "hp_comm_free": (None, [P]),
    "hp_compress_ex": (C.c_int, [P, P, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int, P, C.POINTER(P)]),
    "hp_compress_group": (C.c_int, [P, P, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(P)]),
    "hp_shard_owners": (C.c_int, [P, C.c_int, ip, ip, lp]),
    "hp_shard_memory_plan": (C.c_int, [P, C.c_int, C.c_int, C.c_int, dp]),
    "hp_shard_exchange_counts": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, lp, lp]),
    "hp_export_sizes_shard": (C.c_int, [P, C.c_int, C.c_int, C.c_int, lp, lp]),
    "hp_rep_shard": (C.c_int, [P, C.c_int, i64, ip, ip, ip]),
    "hp_partition_ranges": (C.c_int, [dp, i64, C.c_int, lp]),
    "hp_rep_report": (C.c_int, [P, dp, lp]),
    "hp_rep_phase": (C.c_int, [P, i64, lp, dp]),
    "hp_rep_csv": (C.c_int, [P, C.c_char_p, i64, lp]),
    "hp_rep_num_pairs": (C.c_int, [P, C.c_int, lp]),
    "hp_rep_block": (C.c_int, [P, C.c_int, i64, ip, ip, dp, dp, dp]),
    "hp_rep_dense_block": (C.c_int, [P, i64, dp]),
    "hp_rep_apply": (C.c_int, [P, C.c_int, dp, i64, dp]),
    "hp_rep_storage": (C.c_int, [P, lp]),
    "hp_rep_sizes": (C.c_int, [P, lp, lp]),
    "hp_rep_export": (C.c_int, [P, dp, dp, lp]),
    "hp_export_sizes": (C.c_int, [P, C.c_int, lp, lp]),
    "hp_host_alloc": (C.c_int, [i64, C.POINTER(P)]),
    "hp_host_free": (None, [P]),
    "hp_compress_export": (C.c_int, [P, P, C.c_int, C.c_int, u64, C.c_int, C.c_int, P, dp, i64, dp, i64,
                                     C.POINTER(P)]),
    "hp_rep_save": (C.c_int, [P, C.c_char_p]),
    "hp_rep_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(P), C.POINTER(P)]),
    "hp_save_dense_matrix": (C.c_int, [C.c_char_p, dp, i64, i64]),
    "hp_load_dense_matrix": (C.c_int, [C.c_char_p, lp, lp, dp, i64]),
    "hp_rep_captured": (C.c_int, [P, C.c_int, i64, lp, lp, dp]),
    "hp_rep_captured_raw": (C.c_int, [P, C.c_int, i64, lp, lp, dp]),
    "hp_rel_error_power_method": (C.c_int, [P, P, C.c_int, u64, dp]),
}

# probe entry points (paper_2205_03406_b200/csrc/hpeel_probe.h): tests and
# profiling tools only, not part of the drop-in boundary
_PROBE_SIGNATURES = {
    "hp_debug_set_k2_mode": (None, [C.c_int]),
    "hp_debug_set_k2_path": (None, [C.c_int]),
    "hp_debug_payload": (C.c_int, [P, C.c_int, C.c_int, u64, C.c_int, dp]),
    "hp_debug_qr": (C.c_int, [dp, ip, C.c_int, C.c_int, C.c_int, C.c_int, dp, ip, dp]),
    "hp_debug_log": (C.c_int, [dp, i64, C.c_int, dp]),
}

# hp_apply_fn (include/hpeel_b200.h): ctx, adjoint, x, w, y, stream
APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double),
                       C.c_void_p)


def lib():
    """Load the C ABI library (once); raise loudly if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback for the hpeel_b200 path)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in list(_SIGNATURES.items()) + list(_PROBE_SIGNATURES.items()):
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


def probe_symbols():
    return list(_PROBE_SIGNATURES)


def check(rc):
    if rc == HP_OK:
        return
    msg = lib().hp_last_error().decode(errors="replace")
    if rc == HP_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == HP_ERR_LOGIC:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(ip)


def lptr(a: np.ndarray):
    return a.ctypes.data_as(lp)


def fmat(x) -> np.ndarray:
    """Column-major float64 copy (Eigen::MatrixXd layout)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    return np.asfortranarray(x)
