"""Two ranks of the query-sharded engine: on one GPU with gloo carrying the
collectives, and on two GPUs over NCCL (the product path; skipped unless two
devices are visible).  Snapshot
slices and per-tick update slices are all-gathered, every rank re-indexes
the replicated snapshot and answers its query shard, distance_evals are
all-reduced into every rank's rebuild history (sharded.py).
The concatenated rank outputs must equal one engine over all queries."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1412_6170_b200 import Engine, EngineConfig, synth  # noqa: E402
from paper_1412_6170_b200.sharded import ShardedEngine, shard_bounds, shard_queries  # noqa: E402

N, NQ, K, TICKS = 60_000, 6_000, 16, 4


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    snap = synth.place(N, "gaussian", seed=21, hotspots=6, sigma=800.0)
    ups = [synth.updates(snap, 0.1, t, seed=21) for t in range(TICKS)]
    qs = [synth.queries(snap, NQ, seed=30 + t) for t in range(TICKS)]
    return snap, ups, qs


def _rank(rank, world, port, ret, backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    local = rank if backend == "nccl" else 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        snap, ups, qs = _inputs()
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
        eng = ShardedEngine(EngineConfig(k=K, region=synth.REGION), local)
        lo, hi = shard_bounds(N, world, rank)
        out = []
        # tick 0: full snapshot slices; then delta ticks with update slices
        for t in range(TICKS):
            qi, qx, qy = qs[t]
            sel = shard_queries(qi, world, rank)
            if t == 0:
                res = eng.process_tick(snap.ids[lo:hi], snap.x[lo:hi], snap.y[lo:hi], qi[sel],
                                       qx[sel], qy[sel], n_total=N)
                eng.load_slices(T(snap.ids[lo:hi]), T(snap.x[lo:hi]), T(snap.y[lo:hi]))
            else:
                uid, ux, uy = ups[t]
                ulo, uhi = shard_bounds(len(uid), world, rank)
                # odd ticks: slice sizes from shard_bounds; even: exchanged
                res = eng.update_tick(uid[ulo:uhi], ux[ulo:uhi], uy[ulo:uhi], qi[sel], qx[sel],
                                      qy[sel], n_total=len(uid) if t % 2 else None)
            out.append((res.query_ids, res.lengths, res.neighbour_ids, res.distances,
                        eng.job_distance_evals, eng.last_metrics.rebuild_flag))
        eng.close()
        ret[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_two_ranks_equal_one_engine(backend):
    world = 2
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL path needs two visible GPUs")
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_rank, args=(world, _port(), ret, backend), nprocs=world, join=True)
        ranks = [ret[r] for r in range(world)]
    snap, ups, qs = _inputs()
    with Engine(EngineConfig(k=K, region=synth.REGION)) as one:
        for t in range(TICKS):
            if t:
                synth.apply_updates(snap, *ups[t])
            qi, qx, qy = qs[t]
            want = one.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
            for j, arr in enumerate((want.query_ids, want.lengths, want.neighbour_ids)):
                got = np.concatenate([r[t][j] for r in ranks])
                bad = np.nonzero(got != arr)[0]
                assert len(bad) == 0, (t, j, len(bad), bad[:5], got[bad[:5]], arr[bad[:5]])
            got_d = np.concatenate([r[t][3] for r in ranks])
            assert got_d.tobytes() == want.distances.tobytes()
            # job-wide distance_evals (the rebuild history input) == one engine's
            assert ranks[0][t][4] == ranks[1][t][4] == one.last_metrics.distance_evals
            assert ranks[0][t][5] == ranks[1][t][5] == one.last_metrics.rebuild_flag
