"""ctypes binding of libmknn_b200.so (C-ABI in include/mknn_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is usable, calls fail loudly with a RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MKNN_LIB overrides the library path (profiling builds of variants only)
LIB_PATH = os.environ.get("MKNN_LIB") or os.path.join(_HERE, "libmknn_b200.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

EINVAL = -1
ECUDA = -2
EUNSUPPORTED = -3


class Config(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32), ("th_quad", ctypes.c_int32), ("l_max", ctypes.c_int32),
        ("rebuild_window", ctypes.c_int32), ("rebuild_factor", ctypes.c_double),
        ("x_lo", ctypes.c_double), ("y_lo", ctypes.c_double), ("x_hi", ctypes.c_double),
        ("y_hi", ctypes.c_double), ("self_check", ctypes.c_int32),
        ("audit_pruning", ctypes.c_int32), ("device", ctypes.c_int32),
        ("instrument", ctypes.c_int32),
    ]


METRIC_FIELDS = (
    "tick", "n_objects", "n_queries", "iterations_left", "iterations_right", "distance_evals",
    "pruned_leaves", "rebuild_flag", "t_build_us", "t_index_objects_us", "t_index_queries_us",
    "t_first_iteration_us", "t_loop_us", "t_total_us", "pruning_violations", "clamped_objects",
    "n_results", "t_emit_us", "streamed_records",
)


class Metrics(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in METRIC_FIELDS]


# name -> (restype, argtypes); every symbol include/mknn_b200.h declares
SIGNATURES = {
    "mknn_abi_version": (ctypes.c_int, []),
    "mknn_kernel_launches": (ctypes.c_int64, []),
    "mknn_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(_vp)]),
    "mknn_destroy": (None, [_vp]),
    "mknn_last_error": (ctypes.c_char_p, [_vp]),
    "mknn_set_stream": (ctypes.c_int, [_vp, _vp]),
    "mknn_tick": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, ctypes.POINTER(Metrics)]),
    "mknn_tick_device": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64, _vp,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        ctypes.POINTER(Metrics)]),
    "mknn_load": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp]),
    "mknn_update": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp]),
    "mknn_update_device": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp]),
    "mknn_snapshot_size": (ctypes.c_int, [_vp, _i64p]),
    "mknn_query": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  ctypes.POINTER(Metrics)]),
    "mknn_query_device": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                         _vp, ctypes.POINTER(Metrics)]),
    "mknn_set_instrument": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "mknn_graph_stats": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "mknn_set_last_evals": (ctypes.c_int, [_vp, ctypes.c_int64]),
    "mknn_active_counts": (ctypes.c_int64, [_vp, ctypes.c_int, _i64p, ctypes.c_int64]),
    "mknn_index_info": (ctypes.c_int, [_vp, _i32p, _i64p, _i64p, _i64p]),
    "mknn_index_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mknn_store_export": (ctypes.c_int, [_vp, _vp, _vp]),
    "mknn_format_result_rows": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                                 _vp, ctypes.c_int64, ctypes.c_int32]),
    "mknn_bf_count_device": (ctypes.c_int, [ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp,
                                            _vp, _vp, _vp, _vp, _vp]),
}

_lib = None


def lib():
    """Load libmknn_b200.so (built by __graft_entry__.build() / make)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); "
                "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, handle=None, what: str = "") -> None:
    if rc == 0:
        return
    msg = ""
    try:
        m = lib().mknn_last_error(handle)
        msg = m.decode() if m else ""
    except Exception:  # pragma: no cover
        pass
    text = f"{what}: {msg}" if what else msg
    if rc == EINVAL:
        raise ValueError(text or "invalid argument")
    if rc == EUNSUPPORTED:
        raise NotImplementedError(text or "unsupported")
    raise RuntimeError(text or f"mknn error {rc}")
