"""ctypes front end for the C oracle (mknn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg.  The product
package never imports this module.

Each wrapper names the reference function it restates (paths relative to
/root/reference/pkg/src/mknn/).  The restatement is pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Rect(ctypes.Structure):
    _fields_ = [("x_lo", ctypes.c_double), ("y_lo", ctypes.c_double),
                ("x_hi", ctypes.c_double), ("y_hi", ctypes.c_double)]


class _Index(ctypes.Structure):
    _fields_ = [("l_deep", ctypes.c_int32), ("n_leaves", ctypes.c_int64),
                ("overfull", ctypes.c_int64), ("leaf_level", _i32p),
                ("leaf_code", _i64p), ("leaf_key", _i64p), ("leaf_span", _i64p),
                ("build_counts", _i64p), ("z_map", _i32p)]


class _Metrics(ctypes.Structure):
    _fields_ = [("distance_evals", ctypes.c_int64), ("pruned_leaves", ctypes.c_int64),
                ("clamped_objects", ctypes.c_int64), ("iterations_left", ctypes.c_int64),
                ("iterations_right", ctypes.c_int64), ("streamed_records", ctypes.c_int64)]


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_encode.restype = ctypes.c_int64
        L.or_encode.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.POINTER(_Rect), ctypes.c_int]
        L.or_brute_knn.restype = None
        L.or_build_index.restype = ctypes.POINTER(_Index)
        L.or_index_free.restype = None
        L.or_index_objects.restype = ctypes.c_int64
        L.or_engine_tick.restype = ctypes.c_int
        L.or_engine_tick_ix.restype = ctypes.c_int
        L.or_set_num_threads.restype = None
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _rect(region) -> _Rect:
    return _Rect(float(region.x_lo), float(region.y_lo), float(region.x_hi), float(region.y_hi))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


@dataclass
class CSR:
    """Per-query lists in issuer order; same fields as TickResult
    (engine.py:134-156) / OracleResult (oracle.py:22-38)."""

    query_ids: np.ndarray
    lengths: np.ndarray
    offsets: np.ndarray
    neighbour_ids: np.ndarray
    distances: np.ndarray
    metrics: dict = field(default_factory=dict)

    @property
    def n_queries(self) -> int:
        return len(self.query_ids)

    def neighbours(self, i: int):
        s, e = self.offsets[i], self.offsets[i + 1]
        return self.neighbour_ids[s:e], self.distances[s:e]


def _compact(qids, lens, nids, dist, k) -> CSR:
    valid = np.arange(k)[None, :] < lens[:, None]
    offsets = np.concatenate(([0], np.cumsum(lens, dtype=np.int64)))
    return CSR(qids, lens, offsets, nids.reshape(-1, k)[valid], dist.reshape(-1, k)[valid])


def encode(x: float, y: float, region, level: int) -> int:
    """geometry.py:132-135 encode_points for one point."""
    r = _rect(region)
    return int(lib().or_encode(float(x), float(y), ctypes.byref(r), int(level)))


def brute_force_knn(ids, x, y, q_issuer, qx, qy, k: int) -> CSR:
    """oracle.py:41-106 brute_force_knn: canonical (d2, id) lists."""
    ids, x, y = _i64(ids), _f64(x), _f64(y)
    q_issuer, qx, qy = _i64(q_issuer), _f64(qx), _f64(qy)
    n, nq = len(ids), len(q_issuer)
    qids = np.zeros(nq, np.int64)
    lens = np.zeros(nq, np.int32)
    nids = np.zeros(nq * k, np.int64)
    dist = np.zeros(nq * k, np.float64)
    lib().or_brute_knn(
        ctypes.c_int64(n), _p(ids, _i64p), _p(x, _f64p), _p(y, _f64p), ctypes.c_int64(nq),
        _p(q_issuer, _i64p), _p(qx, _f64p), _p(qy, _f64p), ctypes.c_int(k),
        _p(qids, _i64p), _p(lens, _i32p), _p(nids, _i64p), _p(dist, _f64p))
    return _compact(qids, lens, nids, dist, k)


def build_index(x, y, region, th_quad: int, l_max: int) -> dict:
    """quadindex.py:79-163 build_index; returns the QuadIndex arrays."""
    x, y = _f64(x), _f64(y)
    r = _rect(region)
    L = lib()
    p = L.or_build_index(ctypes.c_int64(len(x)), _p(x, _f64p), _p(y, _f64p), ctypes.byref(r),
                         ctypes.c_int(th_quad), ctypes.c_int(l_max))
    if not p:
        raise ValueError(f"bad index parameters th_quad={th_quad} l_max={l_max}")
    ix = p.contents
    m = ix.n_leaves
    out = dict(
        l_deep=int(ix.l_deep), n_leaves=int(m), overfull_leaves=int(ix.overfull),
        leaf_level=np.ctypeslib.as_array(ix.leaf_level, (m,)).copy(),
        leaf_code=np.ctypeslib.as_array(ix.leaf_code, (m,)).copy(),
        leaf_key=np.ctypeslib.as_array(ix.leaf_key, (m,)).copy(),
        leaf_span=np.ctypeslib.as_array(ix.leaf_span, (m,)).copy(),
        build_counts=np.ctypeslib.as_array(ix.build_counts, (m,)).copy(),
        z_map=np.ctypeslib.as_array(ix.z_map, (4 ** int(ix.l_deep),)).copy(),
    )
    out["_ptr"] = p
    return out


def index_objects(ids, x, y, region, index: dict) -> dict:
    """quadindex.py:190-213 index_objects against an oracle index."""
    ids, x, y = _i64(ids), _f64(x), _f64(y)
    n, m = len(ids), index["n_leaves"]
    r = _rect(region)
    s_ids = np.zeros(n, np.int64)
    s_x = np.zeros(n)
    s_y = np.zeros(n)
    cs = np.zeros(m, np.int64)
    ce = np.zeros(m, np.int64)
    clamped = lib().or_index_objects(
        ctypes.c_int64(n), _p(ids, _i64p), _p(x, _f64p), _p(y, _f64p), ctypes.byref(r),
        index["_ptr"], _p(s_ids, _i64p), _p(s_x, _f64p), _p(s_y, _f64p),
        _p(cs, _i64p), _p(ce, _i64p))
    return dict(ids=s_ids, x=s_x, y=s_y, cell_start=cs, cell_end=ce, clamped=int(clamped))


def free_index(index: dict) -> None:
    p = index.pop("_ptr", None)
    if p:
        lib().or_index_free(p)


def engine_tick(ids, x, y, q_issuer, qx, qy, k: int, region, th_quad: int,
                l_max: int = 10, build_xy=None, index: dict | None = None) -> CSR:
    """engine.py:601-696 process_tick with canonical selection.

    The index is built from ``build_xy`` = (bx, by) -- the positions of the
    tick that last rebuilt -- or from this tick's positions when None; or,
    with ``index`` (a ``build_index`` result), that index is reused as on a
    tick where should_rebuild does not fire (engine.py:615-619).

    metrics holds distance_evals, pruned_leaves, clamped_objects,
    iterations_left/right and active_left/right (engine.py:88-107).
    """
    ids, x, y = _i64(ids), _f64(x), _f64(y)
    q_issuer, qx, qy = _i64(q_issuer), _f64(qx), _f64(qy)
    n, nq = len(ids), len(q_issuer)
    r = _rect(region)
    qids = np.zeros(nq, np.int64)
    lens = np.zeros(nq, np.int32)
    nids = np.zeros(nq * k, np.int64)
    dist = np.zeros(nq * k, np.float64)
    navl = np.zeros(nq, np.int32)
    navr = np.zeros(nq, np.int32)
    met = _Metrics()
    l_deep = ctypes.c_int32(0)
    n_leaves = ctypes.c_int64(0)
    head = (ctypes.c_int64(n), _p(ids, _i64p), _p(x, _f64p), _p(y, _f64p), ctypes.c_int64(nq),
            _p(q_issuer, _i64p), _p(qx, _f64p), _p(qy, _f64p), ctypes.c_int(k), ctypes.byref(r))
    outs = (_p(qids, _i64p), _p(lens, _i32p), _p(nids, _i64p), _p(dist, _f64p),
            _p(navl, _i32p), _p(navr, _i32p), ctypes.byref(met), ctypes.byref(l_deep),
            ctypes.byref(n_leaves))
    if index is not None:
        rc = lib().or_engine_tick_ix(*head, index["_ptr"], *outs)
    else:
        bx, by = (x, y) if build_xy is None else (_f64(build_xy[0]), _f64(build_xy[1]))
        rc = lib().or_engine_tick(*head, ctypes.c_int(th_quad), ctypes.c_int(l_max), *outs,
                                  ctypes.c_int64(len(bx)), _p(bx, _f64p), _p(by, _f64p))
    if rc != 0:
        raise ValueError(f"bad index parameters th_quad={th_quad} l_max={l_max}")
    res = _compact(qids, lens, nids, dist, k)
    res.metrics = dict(
        distance_evals=int(met.distance_evals), pruned_leaves=int(met.pruned_leaves),
        clamped_objects=int(met.clamped_objects), iterations_left=int(met.iterations_left),
        iterations_right=int(met.iterations_right),
        streamed_records=int(met.streamed_records),
        active_left=active_counts(navl), active_right=active_counts(navr),
        l_deep=int(l_deep.value), n_leaves=int(n_leaves.value))
    return res


def active_counts(nav_calls: np.ndarray) -> list:
    """engine.py:661-663: refs alive at each same-direction iteration i are
    the queries with more than i navigate calls in that direction."""
    if nav_calls.size == 0:
        return []
    h = np.bincount(nav_calls)
    alive = h[::-1].cumsum()[::-1]  # alive[i] = #{calls >= i}
    return [int(v) for v in alive[1:]]


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the port's query loop (BASELINE.md §3 asks for
    threads=1 and threads=os.cpu_count())."""
    lib().or_set_num_threads(ctypes.c_int(int(n)))
