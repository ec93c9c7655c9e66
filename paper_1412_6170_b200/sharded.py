"""Query-sharded multi-GPU ticks.

One process per GPU (torchrun), ``torch.distributed`` over NCCL for the
plumbing.  Per tick:

1. each rank holds a 1/G slice of the position snapshot or of the tick's
   update records (24 B each: int64 id, f64 x, f64 y);
2. the slices are all-gathered over NVLink/NVSwitch (three
   ``all_gather_into_tensor`` calls, one per column, so the gathered columns
   are contiguous and feed the engine without a repack);
3. every rank rebuilds / re-indexes the replicated index and answers its own
   query shard (contiguous issuer-id range, so the per-rank CSR outputs
   concatenate in issuer order);
4. the per-tick ``distance_evals`` are all-reduced and written back into each
   rank's rebuild history (``mknn_set_last_evals``), so every rank takes the
   reference's rebuild decision (quadindex.py:231-246) on the job-wide count.

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


def all_gather_columns(cols, group=None):
    """All-gather equally-typed 1-D tensors whose lengths may differ per rank.

    Returns the concatenation over ranks (rank order) of each column.  Lengths
    are exchanged first; slices are padded to the longest one and the padding
    is dropped after the gather.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = cols[0].device
    n_local = torch.tensor([cols[0].numel()], dtype=torch.int64, device=dev)
    sizes = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, n_local, group=group)
    sizes_h = sizes.cpu().tolist()
    width = max(sizes_h) if sizes_h else 0
    out = []
    for c in cols:
        if c.numel() < width:
            pad = torch.zeros(width - c.numel(), dtype=c.dtype, device=dev)
            c = torch.cat([c, pad])
        g = torch.empty(world * width, dtype=c.dtype, device=dev)
        dist.all_gather_into_tensor(g, c.contiguous(), group=group)
        if any(s != width for s in sizes_h):
            g = torch.cat([g[r * width: r * width + s] for r, s in enumerate(sizes_h)])
        out.append(g)
    return out


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

    def close(self) -> None:
        self.engine.close()

    def _reduce_evals(self) -> None:
        import torch.distributed as dist

        torch = self.torch
        m = self.engine.last_metrics
        t = torch.tensor([m.distance_evals], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, group=self.group)
        total = int(t.item())
        N.check(N.lib().mknn_set_last_evals(self.engine._h, total), self.engine._h)
        self.job_distance_evals = total
        self.last_metrics = m

    def load_slices(self, ids_s, x_s, y_s) -> None:
        """Initial device-resident snapshot from per-rank slices (device
        tensors): the gathered columns are applied as updates to every rank's
        empty snapshot (new ids are appended, datasets.py:136-148)."""
        ids, x, y = all_gather_columns([ids_s, x_s, y_s], self.group)
        self.engine.update(ids, x, y)

    def update_tick_device(self, u_ids_s, ux_s, uy_s, q_issuer, qx, qy, out=None):
        """Delta tick: every rank holds 1/G of the tick's position updates
        (24-byte records); they are all-gathered over NCCL, applied to every
        rank's replicated snapshot (last update per id wins) and the rank's
        query shard is answered over it."""
        ids, x, y = all_gather_columns([u_ids_s, ux_s, uy_s], self.group)
        self.engine.update(ids, x, y)
        out = self.engine.query_device(q_issuer, qx, qy, out=out)
        self._reduce_evals()
        return out

    def update_tick(self, u_ids_s, ux_s, uy_s, q_issuer, qx, qy) -> TickResult:
        """Delta tick with host arrays in (this rank's update slice and query
        shard) and a host TickResult out (this rank's rows, issuer order)."""
        torch = self.torch
        dev = self.device

        def h2d(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev, non_blocking=True)

        out = self.update_tick_device(h2d(u_ids_s, np.int64), h2d(ux_s, np.float64),
                                      h2d(uy_s, np.float64), h2d(q_issuer, np.int64),
                                      h2d(qx, np.float64), h2d(qy, np.float64))
        return self._host_result(out, int(np.asarray(q_issuer).size))

    def _host_result(self, out, nq: int) -> TickResult:
        nres = out["n_results"]
        return TickResult(query_ids=out["query_ids"][:nq].cpu().numpy(),
                          lengths=out["lengths"][:nq].cpu().numpy(),
                          offsets=out["offsets"][: nq + 1].cpu().numpy(),
                          neighbour_ids=out["neighbour_ids"][:nres].cpu().numpy(),
                          distances=out["distances"][:nres].cpu().numpy())

    def tick_device(self, ids_s, x_s, y_s, q_issuer, qx, qy, out=None):
        """Snapshot slices + this rank's queries, all CUDA tensors; results
        stay on the device (Engine.tick_device layout)."""
        ids, x, y = all_gather_columns([ids_s, x_s, y_s], self.group)
        out = self.engine.tick_device(ids, x, y, q_issuer, qx, qy, out=out)
        self._reduce_evals()
        return out

    def process_tick(self, ids_s, x_s, y_s, q_issuer, qx, qy) -> TickResult:
        """Host arrays in (this rank's snapshot slice and query shard), host
        TickResult out (this rank's rows, in issuer order)."""
        torch = self.torch
        dev = self.device

        def h2d(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev, non_blocking=True)

        out = self.tick_device(h2d(ids_s, np.int64), h2d(x_s, np.float64), h2d(y_s, np.float64),
                               h2d(q_issuer, np.int64), h2d(qx, np.float64), h2d(qy, np.float64))
        return self._host_result(out, int(np.asarray(q_issuer).size))
