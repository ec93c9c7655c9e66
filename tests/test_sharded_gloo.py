"""World-size-2 gloo tests of the multi-GPU host logic (sharded.py) on CPU.

The data-path collective (all-gather of snapshot / update slices) and the
query sharding run here with CPU tensors; the per-rank k-NN answer is the
oracle (the checker), so the test proves that rank outputs concatenate into
exactly the single-process result (engine.py:713 row order) and that the
rebuild-history reduction sees the job-wide distance_evals.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_6170_b200.sharded import all_gather_records, shard_bounds, shard_queries


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 10, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_queries_concatenate_in_stable_issuer_order():
    rng = np.random.default_rng(1)
    qi = rng.integers(0, 50, size=200)  # duplicates: stable order matters
    parts = [shard_queries(qi, 3, r) for r in range(3)]
    cat = np.concatenate(parts)
    assert np.array_equal(cat, np.argsort(qi, kind="stable"))


def _worker(rank, world, port, n, nq, k, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_1412_6170_b200 import synth

        snap = synth.place(n, "gaussian", seed=11, hotspots=4, sigma=900.0)
        qi, qx, qy = synth.queries(snap, nq, seed=11)
        lo, hi = shard_bounds(n, world, rank)
        cols = [torch.from_numpy(snap.ids[lo:hi].copy()), torch.from_numpy(snap.x[lo:hi].copy()),
                torch.from_numpy(snap.y[lo:hi].copy())]
        # sizes known from shard_bounds (no exchange) and exchanged: same records
        ids, x, y = all_gather_records(*cols, n_total=n)
        ids2, x2, y2 = all_gather_records(*cols)
        assert torch.equal(ids, ids2) and torch.equal(x, x2) and torch.equal(y, y2)
        with pytest.raises(ValueError):
            all_gather_records(*cols, n_total=n + 2 * world + 1)
        sel = shard_queries(qi, world, rank)
        res = orc.brute_force_knn(ids.numpy(), x.numpy(), y.numpy(), qi[sel], qx[sel], qy[sel], k)
        evals = torch.tensor([int(res.lengths.sum())], dtype=torch.int64)
        dist.all_reduce(evals)
        ret[rank] = dict(gathered_equal=bool(np.array_equal(ids.numpy(), snap.ids)
                                            and x.numpy().tobytes() == snap.x.tobytes()
                                            and y.numpy().tobytes() == snap.y.tobytes()),
                         qids=res.query_ids, lens=res.lengths, nids=res.neighbour_ids,
                         dist=res.distances, evals=int(evals.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nq", [(3001, 401), (2000, 2)])
def test_two_rank_gather_and_shard_equals_single_process(n, nq):
    world, k = 2, 8
    port = _free_port()
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker, args=(world, port, n, nq, k, ret), nprocs=world, join=True)
        out = [ret[r] for r in range(world)]
    from oracle import oracle as orc
    from paper_1412_6170_b200 import synth

    snap = synth.place(n, "gaussian", seed=11, hotspots=4, sigma=900.0)
    qi, qx, qy = synth.queries(snap, nq, seed=11)
    want = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi, qx, qy, k)
    assert all(o["gathered_equal"] for o in out)
    assert np.array_equal(np.concatenate([o["qids"] for o in out]), want.query_ids)
    assert np.array_equal(np.concatenate([o["lens"] for o in out]), want.lengths)
    assert np.array_equal(np.concatenate([o["nids"] for o in out]), want.neighbour_ids)
    assert np.concatenate([o["dist"] for o in out]).tobytes() == want.distances.tobytes()
    assert out[0]["evals"] == out[1]["evals"] == int(want.lengths.sum())


def _delta_worker(rank, world, port, n, nq, k, ret):
    """ShardedEngine.update_tick_device's host logic on CPU tensors: each rank
    holds 1/G of the tick's updates, they are all-gathered and applied to the
    replicated snapshot (last update per id wins, datasets.py:136-148), and
    the rank answers its query shard over the updated snapshot."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_1412_6170_b200 import synth

        snap = synth.place(n, "uniform", seed=5)
        rows = []
        for tick in range(2):
            uid, ux, uy = synth.updates(snap, 0.1, tick, seed=5)
            lo, hi = shard_bounds(len(uid), world, rank)
            g_id, g_x, g_y = all_gather_records(torch.from_numpy(uid[lo:hi].copy()),
                                                torch.from_numpy(ux[lo:hi].copy()),
                                                torch.from_numpy(uy[lo:hi].copy()), n_total=len(uid))
            assert np.array_equal(g_id.numpy(), uid)
            synth.apply_updates(snap, g_id.numpy(), g_x.numpy(), g_y.numpy())
            qi, qx, qy = synth.queries(snap, nq, seed=tick)
            sel = shard_queries(qi, world, rank)
            res = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi[sel], qx[sel], qy[sel], k)
            rows.append((res.query_ids, res.neighbour_ids, res.distances))
        ret[rank] = rows
    finally:
        dist.destroy_process_group()


def test_two_rank_update_gather_equals_single_process():
    world, n, nq, k = 2, 2500, 300, 5
    port = _free_port()
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_delta_worker, args=(world, port, n, nq, k, ret), nprocs=world, join=True)
        out = [ret[r] for r in range(world)]
    from oracle import oracle as orc
    from paper_1412_6170_b200 import synth

    snap = synth.place(n, "uniform", seed=5)
    for tick in range(2):
        synth.apply_updates(snap, *synth.updates(snap, 0.1, tick, seed=5))
        qi, qx, qy = synth.queries(snap, nq, seed=tick)
        want = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi, qx, qy, k)
        assert np.array_equal(np.concatenate([o[tick][0] for o in out]), want.query_ids)
        assert np.array_equal(np.concatenate([o[tick][1] for o in out]), want.neighbour_ids)
        assert np.concatenate([o[tick][2] for o in out]).tobytes() == want.distances.tobytes()
