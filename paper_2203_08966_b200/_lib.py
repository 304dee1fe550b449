"""ctypes binding of libbh.so (the C-ABI declared in include/bh.h).

This is the reference-side FFI for the hot path: the reference package is
Python, so its natural binding is ctypes.  There is no fallback -- if the
library is missing or no CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbh.so")

BH_OK = 0
BH_BAD_ARG = 1
BH_OUT_OF_DOMAIN = 2
BH_DUPLICATE_KEY = 3
BH_UNSORTED = 4
BH_DEPTH_OVERFLOW = 5
BH_STACK_OVERFLOW = 6
BH_CUDA_ERROR = 7
BH_NCCL_ERROR = 8
BH_NO_TREE = 9
BH_OUT_OF_MEMORY = 10

BH_FP32 = 0
BH_FP64 = 1

#: every symbol include/bh.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "bh_create", "bh_destroy", "bh_last_error", "bh_version", "bh_check",
    "bh_bounds_f32", "bh_bounds_f64", "bh_morton_f32", "bh_morton_f64", "bh_sort", "bh_scan_u32",
    "bh_build_f32", "bh_build_f64", "bh_tree_size", "bh_sim_tree_fits_dev", "bh_set_allow_duplicates", "bh_export_tree",
    "bh_traverse_f32", "bh_traverse_f64", "bh_kick_f32", "bh_drift_f32",
    "bh_kick_f64", "bh_drift_f64", "bh_direct_f64", "bh_potential_f64",
    "bh_sim_load", "bh_sim_forces", "bh_sim_step", "bh_sim_store", "bh_stats_get",
    "bh_sim_begin_step", "bh_sim_prepare", "bh_sim_walk_range", "bh_sim_scatter_work",
    "bh_sim_end_step", "bh_sim_export", "bh_sim_import",
    "bh_sim_ipc_handles", "bh_sim_set_peers", "bh_sim_set_peer_ptrs", "bh_sim_result_ptrs",
    "bh_sim_local_maxabs", "bh_sim_set_R", "bh_sim_sort", "bh_sim_keys", "bh_sim_load_state",
    "bh_sim_build_local", "bh_sim_branch_export", "bh_sim_walk_records", "bh_walk_records_f32",
    "bh_sim_let", "bh_sim_let_pack", "bh_sim_target_boxes", "bh_sim_step_host",
    "bh_walk_records_defer_f32", "bh_walk_records_resume_f32",
    "bh_timing_enable", "bh_timing_reset", "bh_timing_get", "bh_ffma_peak", "bh_dfma_peak", "bh_host_register", "bh_host_unregister",
    "bh_ic_plummer", "bh_host_potential_pairs", "bh_top_tree",
)
BH_SIM_ACC, BH_SIM_WORK, BH_SIM_PREV_WORK, BH_SIM_POS, BH_SIM_VEL, BH_SIM_ID, BH_SIM_KEYS = range(7)
PHASES = ("integrate", "keys", "sort", "permute", "build", "walk", "let")


class BHStats(ctypes.Structure):
    _fields_ = [
        ("n_bodies", ctypes.c_int64),
        ("n_cells", ctypes.c_int64),
        ("max_level", ctypes.c_int64),
        ("pp", ctypes.c_int64),
        ("pc", ctypes.c_int64),
        ("work", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("n_records", ctypes.c_int64),
    ]


class BHError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libbh error {code}: {msg}")
        self.code = code


_lib = None
_lock = threading.Lock()


def _declare(L: ctypes.CDLL) -> None:
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "bh_create": ([ctypes.POINTER(P), I, I], I),
        "bh_destroy": ([P], I),
        "bh_last_error": ([], ctypes.c_char_p),
        "bh_version": ([], I),
        "bh_check": ([P, P], I),
        "bh_bounds_f32": ([P, P, I64, P, P], I),
        "bh_bounds_f64": ([P, P, I64, P, P], I),
        "bh_morton_f32": ([P, P, I64, P, P, P], I),
        "bh_morton_f64": ([P, P, I64, P, P, P], I),
        "bh_sort": ([P, P, I64, P, P, P], I),
        "bh_scan_u32": ([P, P, I64, P, I, P], I),
        "bh_build_f32": ([P, P, I64, P, P], I),
        "bh_build_f64": ([P, P, P, I64, P, P], I),
        "bh_tree_size": ([P, ctypes.POINTER(I64)], I),
        "bh_sim_tree_fits_dev": ([P, P, P], I),
        "bh_set_allow_duplicates": ([P, I], I),
        "bh_export_tree": ([P] + [P] * 9 + [P], I),
        "bh_traverse_f32": ([P, P, I64, D, D, I, P, P, P], I),
        "bh_traverse_f64": ([P, P, I64, D, D, I, P, P, P], I),
        "bh_kick_f32": ([P, P, P, I64, D, P], I),
        "bh_drift_f32": ([P, P, P, I64, D, P], I),
        "bh_kick_f64": ([P, P, P, I64, D, P], I),
        "bh_drift_f64": ([P, P, P, I64, D, P], I),
        "bh_direct_f64": ([P, P, P, I64, D, P, P], I),
        "bh_potential_f64": ([P, P, P, I64, D, P, P], I),
        "bh_sim_load": ([P, P, P, P, P, I64, P], I),
        "bh_sim_forces": ([P, D, D, I, I, P], I),
        "bh_sim_step": ([P, D, D, D, I, I, P], I),
        "bh_sim_store": ([P, P, P, P, P, P], I),
        "bh_stats_get": ([P, ctypes.POINTER(BHStats), P], I),
        "bh_sim_begin_step": ([P, D, P], I),
        "bh_sim_prepare": ([P, D, D, I, I, P], I),
        "bh_sim_walk_range": ([P, D, D, I, I64, I64, I, P], I),
        "bh_sim_scatter_work": ([P, P], I),
        "bh_sim_ipc_handles": ([P, P], I),
        "bh_sim_set_peers": ([P, I, P], I),
        "bh_sim_set_peer_ptrs": ([P, I, P, P], I),
        "bh_sim_result_ptrs": ([P, ctypes.POINTER(P), ctypes.POINTER(P)], I),
        "bh_sim_end_step": ([P, D, P], I),
        "bh_sim_export": ([P, I, I64, I64, P, P], I),
        "bh_sim_import": ([P, I, I64, I64, P, P], I),
        "bh_sim_local_maxabs": ([P, ctypes.POINTER(D), P], I),
        "bh_sim_set_R": ([P, D, P], I),
        "bh_sim_sort": ([P, P], I),
        "bh_sim_keys": ([P, P, P], I),
        "bh_sim_load_state": ([P, P, P, P, P, I64, P], I),
        "bh_sim_build_local": ([P, D, I, I, ctypes.c_uint64, I, ctypes.c_uint64, ctypes.POINTER(I64), P], I),
        "bh_sim_branch_export": ([P, P, P, P, P, P, P, P], I),
        "bh_sim_walk_records": ([P, P, ctypes.POINTER(I64), P], I),
        "bh_walk_records_f32": ([P, P, I64, P, P, I64, D, I, P, P, P], I),
        "bh_sim_let": ([P, P, I, I, I, ctypes.POINTER(I64), ctypes.POINTER(I64), P], I),
        "bh_sim_let_pack": ([P, I, P, P, P, P], I),
        "bh_sim_target_boxes": ([P, P, I, P, P], I),
        "bh_sim_step_host": ([P, P, P, P, P, I64, D, D, D, I, I, P], I),
        "bh_walk_records_defer_f32": ([P, P, I64, P, P, I64, D, I, P, P, P, P, I64, P], I),
        "bh_walk_records_resume_f32": ([P, P, I64, P, P, I64, D, I, P, P, P, I64, P, P], I),
        "bh_timing_enable": ([P, I], I),
        "bh_timing_reset": ([P], I),
        "bh_timing_get": ([P, ctypes.POINTER(D), I], I),
        "bh_ffma_peak": ([P, ctypes.POINTER(D), P], I),
        "bh_host_register": ([P, I64], I),
        "bh_host_unregister": ([P], I),
        "bh_dfma_peak": ([P, ctypes.POINTER(D), P], I),
        "bh_ic_plummer": ([P, I64, I64, D, P, P, ctypes.POINTER(I64)], I64),
        "bh_host_potential_pairs": ([P, P, I64, D], D),
        "bh_top_tree": ([P, I64, I64, I, D, D, P, P, P, P, I64], I64),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """Load libbh.so; raises if it was not built (no silent fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_2203_08966_b200.build_lib` (nvcc, sm_100a)")
            L = ctypes.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().bh_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> None:
    """Map a bh_status to the reference's exception types and messages."""
    if code == BH_OK:
        return
    msg = last_error()
    if code in (BH_OUT_OF_DOMAIN, BH_DUPLICATE_KEY, BH_UNSORTED, BH_DEPTH_OVERFLOW, BH_BAD_ARG):
        raise ValueError(msg)
    raise BHError(code, msg)
