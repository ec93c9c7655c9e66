"""Query-sharded multi-GPU ticks.

One process per GPU (torchrun), ``torch.distributed`` over NCCL for the
plumbing.  Per tick:

1. each rank holds a 1/G slice of the position snapshot or of the tick's
   update records (24 B each: int64 id, f64 x, f64 y);
2. the slices are all-gathered over NVLink/NVSwitch in ONE
   ``all_gather_into_tensor`` of packed 24-byte records; every rank's slice
   size follows from ``shard_bounds`` and the job-wide count, so no size
   exchange (and no host synchronisation) precedes the gather;
3. every rank rebuilds / re-indexes the replicated index and answers its own
   query shard (contiguous issuer-id range, so the per-rank CSR outputs
   concatenate in issuer order);
4. the per-tick ``distance_evals`` are all-reduced (asynchronously) and
   written back into each rank's rebuild history (``mknn_set_last_evals``)
   before the rank's next tick, so every rank takes the reference's rebuild
   decision (quadindex.py:231-246) on the job-wide count.

There is no other data-path collective: queries are independent given the
snapshot.  The host-side logic (slicing, padding, gathering, sharding) is
covered by world-size-2 gloo tests on CPU (tests/test_sharded_gloo.py).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .engine import Engine, EngineConfig, TickResult


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous [lo, hi) slice of n items for one rank (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_queries(q_issuer, world: int, rank: int):
    """Indices of this rank's queries: a contiguous block of the stable
    issuer order, so rank outputs concatenate into the global row order
    (engine.py:713)."""
    order = np.argsort(np.asarray(q_issuer, dtype=np.int64), kind="stable")
    lo, hi = shard_bounds(len(order), world, rank)
    return order[lo:hi]


def _slice_sizes(n_total: int, world: int):
    return [hi - lo for lo, hi in (shard_bounds(n_total, world, r) for r in range(world))]


_KEEP_CACHE: dict = {}


def all_gather_records(ids, x, y, n_total=None, group=None):
    """All-gather this rank's slice of (id, x, y) records in ONE collective.

    The three columns are packed as a [3, width] int64 block (the doubles by
    bit pattern), gathered into [world, 3, width] and unpacked into three
    contiguous columns in rank order.  With ``n_total`` (the job-wide record
    count, sliced by ``shard_bounds``) every rank's size is known locally;
    without it the sizes are exchanged first (one extra collective and a
    host read).  Slices shorter than the widest are padded and the padding
    dropped after the gather.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = ids.device
    n = ids.numel()
    if n_total is None:
        n_local = torch.tensor([n], dtype=torch.int64, device=dev)
        sizes_t = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(sizes_t, n_local, group=group)
        sizes = sizes_t.cpu().tolist()
    else:
        sizes = _slice_sizes(int(n_total), world)
        if sizes[dist.get_rank(group)] != n:
            raise ValueError(f"slice of {n} records is not this rank's shard_bounds slice of "
                             f"{n_total}")
    width = max(sizes) if sizes else 0
    buf = torch.empty((3, width), dtype=torch.int64, device=dev)
    buf[0, :n] = ids
    buf[1, :n] = x.view(torch.int64) if x.dtype == torch.float64 else x.double().view(torch.int64)
    buf[2, :n] = y.view(torch.int64) if y.dtype == torch.float64 else y.double().view(torch.int64)
    if n < width:
        buf[:, n:] = 0
    g = torch.empty((world * 3, width), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(g, buf, group=group)
    cols = g.view(world, 3, width).permute(1, 0, 2).reshape(3, world * width)  # one copy kernel
    if any(s != width for s in sizes):
        key = (tuple(sizes), str(dev))
        keep = _KEEP_CACHE.get(key)
        if keep is None:
            keep = torch.cat([torch.arange(r * width, r * width + s, device=dev)
                              for r, s in enumerate(sizes)])
            _KEEP_CACHE[key] = keep
        cols = cols[:, keep]
    return cols[0], cols[1].view(torch.float64), cols[2].view(torch.float64)


class ShardedEngine:
    """Replicated-index, query-sharded engine for one rank of a torchrun job."""

    def __init__(self, config: EngineConfig, local_rank: int, group=None):
        import torch

        self.torch = torch
        self.group = group
        self.device = torch.device("cuda", local_rank)
        config.device = local_rank
        self.engine = Engine(config)
        self.engine.set_stream(torch.cuda.current_stream(self.device))
        self.last_metrics = None
        self._pending_evals = None  # all-reduced distance_evals not yet applied
        self._job_evals = 0

    def close(self) -> None:
        self.engine.close()

    def _reduce_evals(self) -> None:
        """Enqueue the all-reduce of this tick's distance_evals; it is read
        (and written into the rebuild history) before the next tick."""
        import torch.distributed as dist

        torch = self.torch
        m = self.engine.last_metrics
        t = torch.tensor([m.distance_evals], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, group=self.group)
        self._pending_evals = t
        self.last_metrics = m

    def _apply_pending(self) -> None:
        t = self._pending_evals
        if t is None:
            return
        self._pending_evals = None
        total = int(t.item())
        N.check(N.lib().mknn_set_last_evals(self.engine._h, total), self.engine._h)
        self._job_evals = total

    @property
    def job_distance_evals(self) -> int:
        """Job-wide distance_evals of the last tick (all ranks)."""
        self._apply_pending()
        return self._job_evals

    def load_slices(self, ids_s, x_s, y_s, n_total=None) -> None:
        """Initial device-resident snapshot from per-rank slices (device
        tensors): the gathered records are applied as updates to every rank's
        empty snapshot (new ids are appended, datasets.py:136-148).
        n_total: the job-wide record count (slices by shard_bounds)."""
        ids, x, y = all_gather_records(ids_s, x_s, y_s, n_total, self.group)
        self.engine.update(ids, x, y)

    def update_tick_device(self, u_ids_s, ux_s, uy_s, q_issuer, qx, qy, out=None, n_total=None):
        """Delta tick: every rank holds 1/G of the tick's position updates
        (24-byte records); they are all-gathered over NCCL, applied to every
        rank's replicated snapshot (last update per id wins) and the rank's
        query shard is answered over it.  n_total: the
        tick's job-wide update count (slices by shard_bounds)."""
        ids, x, y = all_gather_records(u_ids_s, ux_s, uy_s, n_total, self.group)
        self._apply_pending()
        self.engine.update(ids, x, y)
        out = self.engine.query_device(q_issuer, qx, qy, out=out)
        self._reduce_evals()
        return out

    def update_tick(self, u_ids_s, ux_s, uy_s, q_issuer, qx, qy, n_total=None) -> TickResult:
        """Delta tick with host arrays in (this rank's update slice and query
        shard) and a host TickResult out (this rank's rows, issuer order)."""
        torch = self.torch
        dev = self.device

        def h2d(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev, non_blocking=True)

        out = self.update_tick_device(h2d(u_ids_s, np.int64), h2d(ux_s, np.float64),
                                      h2d(uy_s, np.float64), h2d(q_issuer, np.int64),
                                      h2d(qx, np.float64), h2d(qy, np.float64), n_total=n_total)
        return self._host_result(out, int(np.asarray(q_issuer).size))

    def _host_result(self, out, nq: int) -> TickResult:
        nres = out["n_results"]
        return TickResult(query_ids=out["query_ids"][:nq].cpu().numpy(),
                          lengths=out["lengths"][:nq].cpu().numpy(),
                          offsets=out["offsets"][: nq + 1].cpu().numpy(),
                          neighbour_ids=out["neighbour_ids"][:nres].cpu().numpy(),
                          distances=out["distances"][:nres].cpu().numpy())

    def tick_device(self, ids_s, x_s, y_s, q_issuer, qx, qy, out=None, n_total=None):
        """Snapshot slices + this rank's queries, all CUDA tensors; results
        stay on the device (Engine.tick_device layout).  n_total: the job-wide
        object count (slices by shard_bounds)."""
        ids, x, y = all_gather_records(ids_s, x_s, y_s, n_total, self.group)
        self._apply_pending()
        out = self.engine.tick_device(ids, x, y, q_issuer, qx, qy, out=out)
        self._reduce_evals()
        return out

    def process_tick(self, ids_s, x_s, y_s, q_issuer, qx, qy, n_total=None) -> TickResult:
        """Host arrays in (this rank's snapshot slice and query shard), host
        TickResult out (this rank's rows, in issuer order)."""
        torch = self.torch
        dev = self.device

        def h2d(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev, non_blocking=True)

        out = self.tick_device(h2d(ids_s, np.int64), h2d(x_s, np.float64), h2d(y_s, np.float64),
                               h2d(q_issuer, np.int64), h2d(qx, np.float64), h2d(qy, np.float64),
                               n_total=n_total)
        return self._host_result(out, int(np.asarray(q_issuer).size))
