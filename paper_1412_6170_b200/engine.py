"""Drop-in tick API of the reference engine, backed by sm_100a kernels.

Mirrors reference pkg/src/mknn/engine.py: ``resolve_th_quad`` (48-56),
``EngineConfig`` (59-85), ``TickMetrics`` (88-131), ``TickResult``
(134-156) and ``Engine`` (557-701) keep their names, fields, argument
meaning and ValueError behaviour.  ``Engine.process_tick`` crosses into
libmknn_b200.so once per tick (include/mknn_b200.h ``mknn_tick``); all index,
search and emission work runs on the GPU.  There is no CPU fallback.

Differences from the reference, all documented in DESIGN.md:
* neighbour ids inside a boundary tie group are the canonical lowest ids
  (the reference oracle's answer, oracle.py:76-90) rather than the
  reference engine's scan-order pick; distances are identical;
* rows of duplicate issuer ids keep input order (oracle.py:56);
* ``num_bins``, ``max_refine_iters`` and ``threads`` configure CPU internals
  and are accepted but unused; ``device`` selects the CUDA ordinal.

Extensions beyond the reference API: ``load`` / ``update`` / ``query`` (the
delta path over a device-resident snapshot, datasets.py:136-148 semantics)
and ``tick_device`` / ``query_device`` (torch CUDA tensors in and out).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .geometry import Rect
from .index import MAX_L_MAX, QuadIndex


def resolve_th_quad(th_quad, k: int) -> int:
    """Leaf capacity: explicit value, or the k-dependent default (engine.py:48-56)."""
    if th_quad != "auto":
        return int(th_quad)
    if k < 32:
        return 192
    if k <= 128:
        return 12 * k
    return 2048


@dataclass
class EngineConfig:
    k: int
    region: Rect
    th_quad: int | str = "auto"
    l_max: int = 10
    num_bins: int = 32
    max_refine_iters: int = 64
    rebuild_window: int = 3
    rebuild_factor: float = 1.5
    threads: int = 1
    self_check: bool = False
    audit_pruning: bool = False
    device: int = 0

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError(f"k must be >= 1, got {self.k}")
        if self.num_bins < 2:
            raise ValueError("num_bins must be >= 2")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.rebuild_window < 1:
            raise ValueError("rebuild_window must be >= 1")
        if self.rebuild_factor <= 0:
            raise ValueError("rebuild_factor must be > 0")
        resolve_th_quad(self.th_quad, self.k)


@dataclass
class TickMetrics:
    tick: int
    n_objects: int
    n_queries: int
    iterations_left: int = 0
    iterations_right: int = 0
    distance_evals: int = 0
    pruned_leaves: int = 0
    rebuild_flag: int = 0
    t_build_us: int = 0
    t_index_objects_us: int = 0
    t_index_queries_us: int = 0
    t_first_iteration_us: int = 0
    t_loop_us: int = 0
    t_total_us: int = 0
    active_left: list = field(default_factory=list)
    active_right: list = field(default_factory=list)
    pruning_violations: int = 0
    clamped_objects: int = 0
    t_emit_us: int = 0

    CSV_FIELDS = (
        "tick", "n_objects", "n_queries", "iterations_left", "iterations_right",
        "distance_evals", "pruned_leaves", "rebuild_flag", "t_build_us", "t_index_objects_us",
        "t_index_queries_us", "t_first_iteration_us", "t_loop_us", "t_total_us",
    )

    @classmethod
    def csv_header(cls) -> str:
        return ",".join(cls.CSV_FIELDS)

    def csv_row(self) -> str:
        return ",".join(str(getattr(self, f)) for f in self.CSV_FIELDS)


@dataclass
class TickResult:
    """Neighbour lists for one tick, sorted by query id; each list sorted by
    (distance, neighbour id) (engine.py:134-156)."""

    query_ids: np.ndarray
    lengths: np.ndarray
    offsets: np.ndarray
    neighbour_ids: np.ndarray
    distances: np.ndarray

    @property
    def n_queries(self) -> int:
        return len(self.query_ids)

    def neighbours(self, i: int):
        s, e = self.offsets[i], self.offsets[i + 1]
        return self.neighbour_ids[s:e], self.distances[s:e]

    def iter_rows(self):
        for i in range(self.n_queries):
            ids, dists = self.neighbours(i)
            yield int(self.query_ids[i]), ids, dists


def _ptr(a) -> int:
    return a.ctypes.data if a.size else 0


def _tptr(t) -> int:
    return t.data_ptr() if t is not None and t.numel() else 0


def _dev(t, dtype, name: str):
    """A device input as a torch CUDA tensor: torch tensors as they are,
    any other DLPack producer (CuPy, JAX, numba, ...) zero-copy through
    torch.from_dlpack; the dtype and layout the C-ABI reads are checked."""
    import torch

    if not isinstance(t, torch.Tensor):
        if not hasattr(t, "__dlpack__"):
            raise TypeError(f"{name}: expected a CUDA tensor or a DLPack device array")
        t = torch.from_dlpack(t)
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous() or t.dim() != 1:
        raise TypeError(f"{name}: expected a contiguous 1-D CUDA {dtype} array, "
                        f"got {t.dtype} {tuple(t.shape)} on {t.device}")
    return t


def _on_cuda(a) -> bool:
    """A CUDA device array (torch, or a DLPack producer on kDLCUDA /
    kDLCUDAManaged)?"""
    if hasattr(a, "is_cuda"):
        return bool(a.is_cuda)
    dd = getattr(a, "__dlpack_device__", None)
    return dd is not None and int(dd()[0]) in (2, 13)


def _dev_xy(ids, x, y):
    import torch

    return (_dev(ids, torch.int64, "ids"), _dev(x, torch.float64, "x"),
            _dev(y, torch.float64, "y"))


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy NULL stream as a handle

_POOL = None


def _host_out(nq: int, k: int):
    """Fresh result arrays for a host tick, owned by the caller (engine.py's
    TickResult arrays are new per tick).  They are page-locked so the
    library's per-slice device->host copies run asynchronously and overlap
    the next slice's search: a copy into pageable memory blocks the host
    until it completes.  torch's pinned caching allocator recycles a block
    once every array viewing it is gone, so steady-state ticks allocate no
    new page-locked memory; without CUDA (never on the product path, which
    needs a device) plain arrays are returned."""
    try:
        import torch

        if torch.cuda.is_available():
            def pinned(n, dt):
                return torch.empty(max(n, 1), dtype=dt, pin_memory=True).numpy()[:n]

            return (pinned(nq, torch.int64), pinned(nq, torch.int32), pinned(nq * k, torch.int64),
                    pinned(nq * k, torch.float64))
    except ImportError:  # pragma: no cover - torch is part of the runtime
        pass
    return (np.empty(nq, np.int64), np.empty(nq, np.int32), np.empty(nq * k, np.int64),
            np.empty(nq * k, np.float64))


def _parallel_fill(fn, n: int, min_chunk: int = 1 << 17) -> None:
    """fn(lo, hi) over [0, n) in chunks on a small thread pool (numpy
    releases the GIL): the 8 MB offsets array of a 1M-query tick costs ~1 ms
    on one host core, most of the host time outside the C call."""
    global _POOL
    parts = min(8, max(1, n // min_chunk))
    if parts == 1:
        fn(0, n)
        return
    if _POOL is None:
        import concurrent.futures

        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=8)
    step = (n + parts - 1) // parts
    list(_POOL.map(lambda i: fn(i * step, min(n, (i + 1) * step)), range(parts)))


class Engine:
    """Stateful tick processor: owns the device index, the rebuild history
    and the device buffers.  Feed it one deduplicated batch per tick."""

    def __init__(self, config: EngineConfig):
        self.config = config
        self.th_quad = resolve_th_quad(config.th_quad, config.k)
        self.last_metrics: TickMetrics | None = None
        self._h = None
        self._index_cache: QuadIndex | None = None
        self._index_tick = -1
        # count the reference's streamed records T per tick (measurement only)
        self._instrument = False
        self.last_streamed_records = -1
        self._user_stream = False
        self._bound_stream = 0
        self._ramp = np.zeros(0, np.int64)  # 0..nq, reused for full-row CSR offsets
        self._act_buf = None  # active-count readback buffer (_finish)
        self._act_ptr = None

    # -- lifecycle (engine.py:570-585) --------------------------------------
    def _handle(self):
        if self._h is None:
            # build_index's parameter checks surface on first use, as in the
            # reference (quadindex.py:86-89)
            if self.th_quad < 1:
                raise ValueError(f"th_quad must be >= 1, got {self.th_quad}")
            if not 1 <= self.config.l_max <= MAX_L_MAX:
                raise ValueError(f"l_max must be in [1, {MAX_L_MAX}], got {self.config.l_max}")
            r = self.config.region
            cfg = N.Config(
                k=self.config.k, th_quad=self.th_quad, l_max=self.config.l_max,
                rebuild_window=self.config.rebuild_window,
                rebuild_factor=float(self.config.rebuild_factor),
                x_lo=float(r.x_lo), y_lo=float(r.y_lo), x_hi=float(r.x_hi), y_hi=float(r.y_hi),
                self_check=int(bool(self.config.self_check)),
                audit_pruning=int(bool(self.config.audit_pruning)),
                device=int(self.config.device), instrument=int(self._instrument))
            h = ctypes.c_void_p()
            N.check(N.lib().mknn_create(ctypes.byref(cfg), ctypes.byref(h)), None, "mknn_create")
            self._h = h
        return self._h

    def close(self) -> None:
        if self._h is not None:
            N.lib().mknn_destroy(self._h)
            self._h = None

    def __enter__(self) -> "Engine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    @property
    def instrument(self) -> bool:
        return self._instrument

    @instrument.setter
    def instrument(self, on: bool) -> None:
        """Count T on the following ticks; measurement only."""
        self._instrument = bool(on)
        if self._h is not None:
            N.check(N.lib().mknn_set_instrument(self._h, int(self._instrument)), self._h)

    @property
    def graph_stats(self):
        """(captures, replays) of the steady-state tick graph on this engine."""
        c, r = ctypes.c_int64(), ctypes.c_int64()
        N.check(N.lib().mknn_graph_stats(self._handle(), ctypes.byref(c), ctypes.byref(r)), self._h)
        return c.value, r.value

    def set_stream(self, stream) -> None:
        """Run on a torch.cuda.Stream (or a raw cudaStream_t int; 0/None =
        the engine's own stream).  torch's default stream is the legacy NULL
        stream, passed on as cudaStreamLegacy so the engine stays ordered
        with it (the engine's own stream is non-blocking)."""
        raw = getattr(stream, "cuda_stream", stream)
        if hasattr(stream, "cuda_stream") and not raw:
            raw = _CUDA_STREAM_LEGACY
        N.check(N.lib().mknn_set_stream(self._handle(), ctypes.c_void_p(raw or 0)), self._h)
        self._user_stream = True

    def _follow_torch_stream(self, t) -> None:
        """Device-tensor calls run on torch's current stream unless the
        caller chose a stream: the tensors are produced and consumed there,
        so the engine's reads and writes stay stream-ordered with them."""
        if self._user_stream:
            return
        import torch

        raw = torch.cuda.current_stream(t.device).cuda_stream or _CUDA_STREAM_LEGACY
        if raw != self._bound_stream:
            N.check(N.lib().mknn_set_stream(self._handle(), ctypes.c_void_p(raw)), self._h)
            self._bound_stream = raw

    # -- engine.py:587-589 ---------------------------------------------------
    @property
    def index(self) -> QuadIndex | None:
        if self._h is None or self.last_metrics is None:
            return None
        if self._index_cache is not None and self._index_tick == self._last_build_tick:
            return self._index_cache
        L = N.lib()
        l_deep = ctypes.c_int32()
        n_leaves = ctypes.c_int64()
        over = ctypes.c_int64()
        n_build = ctypes.c_int64()
        N.check(L.mknn_index_info(self._h, ctypes.byref(l_deep), ctypes.byref(n_leaves),
                                  ctypes.byref(over), ctypes.byref(n_build)), self._h)
        m = n_leaves.value
        lv = np.empty(m, np.int32)
        lc = np.empty(m, np.int64)
        lk = np.empty(m, np.int64)
        ls = np.empty(m, np.int64)
        bc = np.empty(m, np.int64)
        zm = np.empty(4 ** l_deep.value, np.int32)
        N.check(L.mknn_index_export(self._h, _ptr(lv), _ptr(lc), _ptr(lk), _ptr(ls), _ptr(bc),
                                    _ptr(zm)), self._h)
        self._index_cache = QuadIndex(
            mbr=self.config.region, th_quad=self.th_quad, l_max=self.config.l_max,
            l_deep=l_deep.value, leaf_level=lv, leaf_code=lc, leaf_key=lk, leaf_span=ls,
            z_map=zm, build_counts=bc, n_build=n_build.value, overfull_leaves=over.value)
        self._index_tick = self._last_build_tick
        return self._index_cache

    def cell_ranges(self):
        """(cell_start, cell_end) of the last tick's object store
        (ObjectStore, quadindex.py:180-181)."""
        idx = self.index
        cs = np.empty(idx.n_leaves, np.int64)
        ce = np.empty(idx.n_leaves, np.int64)
        N.check(N.lib().mknn_store_export(self._h, _ptr(cs), _ptr(ce)), self._h)
        return cs, ce

    # -- ticks ---------------------------------------------------------------
    def _finish(self, m: N.Metrics) -> TickMetrics:
        L = N.lib()
        act = []
        if self._act_buf is None:
            self._act_buf = np.empty(256, np.int64)
            self._act_ptr = self._act_buf.ctypes.data_as(N._i64p)
        for d in (0, 1):
            # one call in the common case (<= 256 iterations per direction)
            cnt = L.mknn_active_counts(self._h, d, self._act_ptr, len(self._act_buf))
            if cnt > len(self._act_buf):
                self._act_buf = np.empty(cnt, np.int64)
                self._act_ptr = self._act_buf.ctypes.data_as(N._i64p)
                L.mknn_active_counts(self._h, d, self._act_ptr, cnt)
            act.append(self._act_buf[:cnt].tolist())
        tm = TickMetrics(
            tick=m.tick, n_objects=m.n_objects, n_queries=m.n_queries,
            iterations_left=m.iterations_left, iterations_right=m.iterations_right,
            distance_evals=m.distance_evals, pruned_leaves=m.pruned_leaves,
            rebuild_flag=m.rebuild_flag, t_build_us=m.t_build_us,
            t_index_objects_us=m.t_index_objects_us, t_index_queries_us=m.t_index_queries_us,
            t_first_iteration_us=m.t_first_iteration_us, t_loop_us=m.t_loop_us,
            t_total_us=m.t_total_us, active_left=act[0], active_right=act[1],
            pruning_violations=m.pruning_violations, clamped_objects=m.clamped_objects,
            t_emit_us=m.t_emit_us)
        if m.rebuild_flag:
            self._last_build_tick = m.tick
        self.last_streamed_records = m.streamed_records
        self.last_metrics = tm
        if self.config.self_check and m.rebuild_flag:
            # engine.py:620-621: structural invariants of the rebuilt index
            # (quadindex.py:51-76), AssertionError on violation
            self.index.validate()
        return tm

    def _result(self, qids, lens, nids, dist, n_results, offsets=None) -> TickResult:
        k = self.config.k
        nq = len(lens)
        if offsets is None:
            offsets = np.empty(nq + 1, np.int64)
        if n_results == nq * k:  # every row full: the CSR is the padded rows
            if len(self._ramp) != nq + 1:
                self._ramp = np.arange(nq + 1, dtype=np.int64)
            _parallel_fill(lambda lo, hi: np.multiply(self._ramp[lo:hi], k, out=offsets[lo:hi]),
                           nq + 1)
        else:
            offsets[0] = 0
            np.cumsum(lens, out=offsets[1:])
        return TickResult(query_ids=qids, lengths=lens, offsets=offsets,
                          neighbour_ids=nids[:n_results], distances=dist[:n_results])

    def process_tick(self, ids, x, y, q_issuer, qx, qy, out=None) -> TickResult:
        """engine.py:601-696.  ``out`` optionally supplies (qids, lens, nids,
        dist[, offsets]) host buffers (e.g. pinned) of sizes nq, nq, nq*k, nq*k
        [, nq+1]; the returned TickResult views them."""
        h = self._handle()
        k = self.config.k
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        q_issuer = np.ascontiguousarray(q_issuer, dtype=np.int64)
        qx = np.ascontiguousarray(qx, dtype=np.float64)
        qy = np.ascontiguousarray(qy, dtype=np.float64)
        n, nq = len(ids), len(q_issuer)
        if len(x) != n or len(y) != n or len(qx) != nq or len(qy) != nq:
            raise ValueError("coordinate arrays must match the id arrays in length")
        qids, lens, nids, dist = out[:4] if out is not None else _host_out(nq, k)
        m = N.Metrics()
        N.check(N.lib().mknn_tick(h, n, _ptr(ids), _ptr(x), _ptr(y), nq, _ptr(q_issuer), _ptr(qx),
                                  _ptr(qy), _ptr(qids), _ptr(lens), _ptr(nids), _ptr(dist),
                                  ctypes.byref(m)), h, "mknn_tick")
        self._finish(m)
        offs = out[4] if out is not None and len(out) > 4 else None
        return self._result(qids, lens, nids, dist, m.n_results, offs)

    def process_batch(self, batch) -> TickResult:
        """engine.py:698-701."""
        return self.process_tick(batch.ids, batch.x, batch.y, batch.q_issuer, batch.qx, batch.qy)

    # -- device-resident paths ---------------------------------------------
    def tick_device(self, ids, x, y, q_issuer, qx, qy, out=None):
        """process_tick on torch CUDA tensors; returns a dict of device
        tensors (query_ids, lengths, offsets, neighbour_ids, distances) whose
        CSR arrays are padded to nq*k (first n_results entries valid).
        Inputs may be any DLPack device arrays; the results are torch
        tensors, themselves DLPack producers (``x.__dlpack__()``), so other
        frameworks take them zero-copy."""
        h = self._handle()
        ids, x, y = _dev_xy(ids, x, y)
        q_issuer, qx, qy = _dev_xy(q_issuer, qx, qy)
        self._follow_torch_stream(q_issuer)
        nq = int(q_issuer.numel())
        out = out or self.alloc_device_out(nq, q_issuer.device)
        m = N.Metrics()
        N.check(N.lib().mknn_tick_device(
            h, int(ids.numel()), _tptr(ids), _tptr(x), _tptr(y), nq, _tptr(q_issuer), _tptr(qx),
            _tptr(qy), _tptr(out["query_ids"]), _tptr(out["lengths"]), _tptr(out["offsets"]),
            _tptr(out["neighbour_ids"]), _tptr(out["distances"]), ctypes.byref(m)), h,
            "mknn_tick_device")
        self._finish(m)
        out["n_results"] = m.n_results
        return out

    def alloc_device_out(self, nq: int, device):
        import torch

        k = self.config.k
        return dict(
            query_ids=torch.empty(max(nq, 1), dtype=torch.int64, device=device),
            lengths=torch.empty(max(nq, 1), dtype=torch.int32, device=device),
            offsets=torch.empty(nq + 1, dtype=torch.int64, device=device),
            neighbour_ids=torch.empty(max(nq * k, 1), dtype=torch.int64, device=device),
            distances=torch.empty(max(nq * k, 1), dtype=torch.float64, device=device),
        )

    def load(self, ids, x, y) -> None:
        """Replace the device-resident snapshot (host arrays)."""
        h = self._handle()
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        N.check(N.lib().mknn_load(h, len(ids), _ptr(ids), _ptr(x), _ptr(y)), h, "mknn_load")

    def update(self, ids, x, y) -> None:
        """Position updates: last update per id wins, unseen ids are added,
        everything else carries forward (datasets.py:109-164).  Accepts host
        arrays or torch CUDA tensors."""
        h = self._handle()
        if _on_cuda(ids):
            ids, x, y = _dev_xy(ids, x, y)
            self._follow_torch_stream(ids)
            N.check(N.lib().mknn_update_device(h, int(ids.numel()), _tptr(ids), _tptr(x), _tptr(y)),
                    h, "mknn_update_device")
            return
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        N.check(N.lib().mknn_update(h, len(ids), _ptr(ids), _ptr(x), _ptr(y)), h, "mknn_update")

    @property
    def snapshot_size(self) -> int:
        n = ctypes.c_int64()
        N.check(N.lib().mknn_snapshot_size(self._handle(), ctypes.byref(n)), self._h)
        return n.value

    def query(self, q_issuer, qx, qy, out=None) -> TickResult:
        """One tick of queries over the device-resident snapshot."""
        h = self._handle()
        k = self.config.k
        q_issuer = np.ascontiguousarray(q_issuer, dtype=np.int64)
        qx = np.ascontiguousarray(qx, dtype=np.float64)
        qy = np.ascontiguousarray(qy, dtype=np.float64)
        nq = len(q_issuer)
        qids, lens, nids, dist = out[:4] if out is not None else _host_out(nq, k)
        m = N.Metrics()
        N.check(N.lib().mknn_query(h, nq, _ptr(q_issuer), _ptr(qx), _ptr(qy), _ptr(qids),
                                   _ptr(lens), _ptr(nids), _ptr(dist), ctypes.byref(m)), h,
                "mknn_query")
        self._finish(m)
        offs = out[4] if out is not None and len(out) > 4 else None
        return self._result(qids, lens, nids, dist, m.n_results, offs)

    def query_device(self, q_issuer, qx, qy, out=None):
        """query on device arrays (torch or any DLPack producer); returns the
        device result dict of tick_device."""
        h = self._handle()
        q_issuer, qx, qy = _dev_xy(q_issuer, qx, qy)
        self._follow_torch_stream(q_issuer)
        nq = int(q_issuer.numel())
        out = out or self.alloc_device_out(nq, q_issuer.device)
        m = N.Metrics()
        N.check(N.lib().mknn_query_device(
            h, nq, _tptr(q_issuer), _tptr(qx), _tptr(qy), _tptr(out["query_ids"]),
            _tptr(out["lengths"]), _tptr(out["offsets"]), _tptr(out["neighbour_ids"]),
            _tptr(out["distances"]), ctypes.byref(m)), h, "mknn_query_device")
        self._finish(m)
        out["n_results"] = m.n_results
        return out

    _last_build_tick = -1
