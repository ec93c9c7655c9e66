"""GPU parity: the sm_100a path through the C-ABI against the reference's
golden vectors and the pinned C oracle.

Bar: neighbour ids and fp64 distances bit-identical to the reference oracle
(brute_force_knn, oracle.py:41-106: canonical (d2, id) order); per-tick
metrics (distance_evals, pruned_leaves, iterations, active counts, rebuild
flags, clamped objects) identical to the reference engine on non-degenerate
data; index arrays identical to build_index / index_objects.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1412_6170_b200 import Engine, EngineConfig, Rect, synth
from tests import golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

CASES = G.case_names()
DEGENERATE_TIES = {"hand_collinear_ties", "lattice_shuffled_ids_k8", "lattice_shuffled_ids_k32",
                   "duplicate_coords_k17"}


def assert_same(res, want):
    np.testing.assert_array_equal(res.query_ids, want.query_ids)
    np.testing.assert_array_equal(res.lengths, want.lengths)
    np.testing.assert_array_equal(res.neighbour_ids, want.neighbour_ids)
    assert res.distances.tobytes() == want.distances.tobytes()


def engine_for(case):
    m = case.meta
    return Engine(EngineConfig(k=case.k, region=case.region, th_quad=case.th_quad,
                               l_max=case.l_max, rebuild_window=m["rebuild_window"],
                               rebuild_factor=m["rebuild_factor"]))


@pytest.mark.parametrize("name", CASES)
def test_golden_case(name):
    case = G.load(name)
    with engine_for(case) as eng:
        eng.instrument = True
        for t, tick in enumerate(case.ticks):
            res = eng.process_tick(tick.ids, tick.x, tick.y, tick.qi, tick.qx, tick.qy)
            assert G.result_digest(res) == tick.meta["oracle_digest"], f"tick {t}"
            if tick.has("o_nids"):
                np.testing.assert_array_equal(res.neighbour_ids, tick["o_nids"])
                assert res.distances.tobytes() == tick["o_dist"].tobytes()
            m, want = eng.last_metrics, tick.meta["metrics"]
            assert m.rebuild_flag == want["rebuild_flag"], f"tick {t}"
            assert m.clamped_objects == want["clamped_objects"]
            assert m.n_objects == want["n_objects"] and m.n_queries == want["n_queries"]
            if name not in DEGENERATE_TIES:
                for key in ("distance_evals", "pruned_leaves", "iterations_left",
                            "iterations_right", "active_left", "active_right"):
                    assert getattr(m, key) == want[key], (t, key, getattr(m, key), want[key])
                assert eng.last_streamed_records == want["streamed_records"], t
            ix = eng.index
            wi = tick.meta["index"]
            assert ix.l_deep == wi["l_deep"] and ix.n_leaves == wi["n_leaves"]
            assert ix.overfull_leaves == wi["overfull_leaves"]
            assert G.digest(ix.z_map.astype(np.int32)) == wi["z_map_digest"]
            if tick.has("ix_leaf_level"):
                for key in ("leaf_level", "leaf_code", "leaf_key", "leaf_span", "build_counts"):
                    np.testing.assert_array_equal(getattr(ix, key), tick["ix_" + key], err_msg=key)
                cs, ce = eng.cell_ranges()
                np.testing.assert_array_equal(cs, tick["cell_start"])
                np.testing.assert_array_equal(ce, tick["cell_end"])


def test_cfg1_matches_reference():
    """BASELINE.json configs[0]: uniform 100K, 10K queries, k=8."""
    meta, arrs = G.load_cfg1()
    snap = synth.place(100_000, "uniform", seed=0)
    sel = np.random.default_rng(1).choice(100_000, 10_000, replace=False)
    with Engine(EngineConfig(k=8, region=synth.REGION)) as eng:
        eng.instrument = True
        res = eng.process_tick(snap.ids, snap.x, snap.y, snap.ids[sel], snap.x[sel], snap.y[sel])
        m = eng.last_metrics
        assert eng.index.n_leaves == meta["index"]["n_leaves"]
    assert G.result_digest(res) == meta["oracle_digest"]
    for key in ("distance_evals", "pruned_leaves", "iterations_left", "iterations_right",
                "active_left", "active_right"):
        assert getattr(m, key) == meta["metrics"][key], key
    assert eng.last_streamed_records == meta["metrics"]["streamed_records"]


@pytest.mark.parametrize("k", [1, 2, 5, 8, 16, 31, 32, 33, 64, 100, 128, 129, 200, 256, 300, 512])
def test_random_vs_brute_force(k):
    rng = np.random.default_rng(1000 + k)
    n = int(rng.integers(500, 4000))
    region = Rect.square(1000.0)
    x = rng.uniform(0, 1000.0, n)
    y = rng.uniform(0, 1000.0, n)
    if k % 2:  # clustered + duplicated coordinates
        x[: n // 4] = np.clip(rng.normal(300, 20, n // 4), 0, 1000)
        y[: n // 4] = np.clip(rng.normal(700, 20, n // 4), 0, 1000)
        x[n // 4: n // 4 + 50] = x[:50]
        y[n // 4: n // 4 + 50] = y[:50]
    ids = rng.permutation(n).astype(np.int64) * 5 - 777
    nq = int(rng.integers(50, 600))
    sel = rng.choice(n, nq, replace=False)
    qi, qx, qy = ids[sel], x[sel].copy(), y[sel].copy()
    qx[::7] = rng.uniform(0, 1000, qx[::7].size)  # queries away from their issuer
    qi[::11] = 10 ** 12 + np.arange(qi[::11].size)  # issuers that are not objects
    th = int(rng.choice([8, 32, 64, 128]))
    with Engine(EngineConfig(k=k, region=region, th_quad=th, l_max=int(rng.integers(3, 11)))) as eng:
        res = eng.process_tick(ids, x, y, qi, qx, qy)
    assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, k))


def test_duplicate_issuers_keep_input_order():
    rng = np.random.default_rng(5)
    n = 800
    x = rng.uniform(0, 100, n)
    y = rng.uniform(0, 100, n)
    ids = np.arange(n, dtype=np.int64)
    qi = np.array([5, 3, 5, 9, 3, 5])
    qx = rng.uniform(0, 100, 6)
    qy = rng.uniform(0, 100, 6)
    with Engine(EngineConfig(k=7, region=Rect.square(100.0), th_quad=16)) as eng:
        res = eng.process_tick(ids, x, y, qi, qx, qy)
    assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, 7))


@pytest.mark.parametrize("sliced", [False, True])
def test_issuer_rows_distinct_then_repeated(sliced):
    """Row order (engine.py:713) by the issuer bitmap rank while the issuers
    are distinct; a later batch that repeats an id is redone with the stable
    radix sort (duplicates keep their input order), and distinct batches
    after it stay exact.  The sliced case runs the host tick's row slices."""
    rng = np.random.default_rng(9)
    n = 120_000 if sliced else 6_000
    nq = 70_000 if sliced else 900
    x = rng.uniform(0, 300, n)
    y = rng.uniform(0, 300, n)
    ids = rng.permutation(10 * n).astype(np.int64)[:n] + 17
    with Engine(EngineConfig(k=6, region=Rect.square(300.0), th_quad=24)) as eng:
        for t, dup in enumerate([False, False, True, False, True]):
            sel = rng.choice(n, nq, replace=False)
            qi, qx, qy = ids[sel].copy(), x[sel], y[sel]
            if dup:  # repeat some issuers (different positions)
                qi[1::7] = qi[0:-1:7][: len(qi[1::7])]
            res = eng.process_tick(ids, x, y, qi, qx, qy)
            assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, 6))


def test_delta_path_equals_full_snapshot():
    """load + update + query == process_tick on the carried-forward snapshot
    (datasets.py:136-148)."""
    snap = synth.place(30_000, "uniform", seed=11)
    with Engine(EngineConfig(k=32, region=synth.REGION)) as full, \
            Engine(EngineConfig(k=32, region=synth.REGION)) as delta:
        delta.load(snap.ids, snap.x, snap.y)
        for t in range(4):
            if t:
                uid, ux, uy = synth.updates(snap, 0.1, t, seed=11)
                # duplicate updates inside a batch: the last one wins
                uid = np.concatenate([uid[:100], uid])
                ux = np.concatenate([ux[:100] + 1.0, ux])
                uy = np.concatenate([uy[:100] + 1.0, uy])
                delta.update(uid, ux, uy)
                synth.apply_updates(snap, uid[100:], ux[100:], uy[100:])
            qi, qx, qy = synth.queries(snap, 3000, seed=100 + t)
            a = full.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
            b = delta.query(qi, qx, qy)
            assert_same(b, a)
            assert delta.last_metrics.distance_evals == full.last_metrics.distance_evals
        # unseen ids are appended
        delta.update(np.array([10 ** 9]), np.array([5.0]), np.array([5.0]))
        assert delta.snapshot_size == 30_001


def test_device_tensors_path():
    snap = synth.place(50_000, "gaussian", seed=2, hotspots=4)
    qi, qx, qy = synth.queries(snap, 5000, seed=2)
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    with Engine(EngineConfig(k=16, region=synth.REGION)) as eng:
        host = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        out = eng.tick_device(T(snap.ids), T(snap.x), T(snap.y), T(qi), T(qx), T(qy))
        torch.cuda.synchronize()
    nres = out["n_results"]
    assert np.array_equal(out["query_ids"].cpu().numpy(), host.query_ids)
    assert np.array_equal(out["lengths"].cpu().numpy(), host.lengths)
    assert np.array_equal(out["offsets"].cpu().numpy(), host.offsets)
    assert np.array_equal(out["neighbour_ids"][:nres].cpu().numpy(), host.neighbour_ids)
    assert out["distances"][:nres].cpu().numpy().tobytes() == host.distances.tobytes()


@pytest.mark.parametrize("k", [16, 32])
def test_graph_replay_equals_direct(k):
    """Steady-state device ticks replay a captured CUDA graph: every replay
    -- on new contents of the same input buffers, and on the delta path
    (update + query_device over the engine's snapshot) -- equals the direct
    host path (never graphed) on the same data, results and metrics."""
    rng = np.random.default_rng(11)
    snap = synth.place(60_000, "gaussian", seed=4, hotspots=6)
    qi, qx, qy = synth.queries(snap, 6000, seed=4)
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    d = [T(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
    keys = ("distance_evals", "pruned_leaves", "active_left", "active_right", "rebuild_flag")
    with Engine(EngineConfig(k=k, region=synth.REGION)) as g, \
            Engine(EngineConfig(k=k, region=synth.REGION)) as ref:
        out = None
        x, y = snap.x.copy(), snap.y.copy()
        for t in range(6):
            if t >= 3:  # new positions in the same device buffers
                x = np.clip(x + rng.normal(0, 3.0, len(x)), 0, 22500)
                y = np.clip(y + rng.normal(0, 3.0, len(y)), 0, 22500)
                d[1].copy_(T(x))
                d[2].copy_(T(y))
                qx, qy = x[qi], y[qi]
                d[4].copy_(T(qx))
                d[5].copy_(T(qy))
            out = g.tick_device(*d, out=out)
            torch.cuda.synchronize()
            want = ref.process_tick(snap.ids, x, y, qi, qx, qy)
            nres = out["n_results"]
            assert np.array_equal(out["query_ids"].cpu().numpy(), want.query_ids), t
            assert np.array_equal(out["offsets"].cpu().numpy(), want.offsets), t
            assert np.array_equal(out["neighbour_ids"][:nres].cpu().numpy(), want.neighbour_ids), t
            assert out["distances"][:nres].cpu().numpy().tobytes() == want.distances.tobytes(), t
            for key in keys:
                assert getattr(g.last_metrics, key) == getattr(ref.last_metrics, key), (t, key)
        cap, rep = g.graph_stats
        assert cap >= 1 and rep >= 3, (cap, rep)

    # delta path: 10 % updates per tick re-index in full -> graph replays
    with Engine(EngineConfig(k=k, region=synth.REGION)) as g, \
            Engine(EngineConfig(k=k, region=synth.REGION)) as ref:
        g.load(snap.ids, snap.x, snap.y)
        x, y = snap.x.copy(), snap.y.copy()
        qd = [T(a) for a in (qi, snap.x[qi], snap.y[qi])]
        out = None
        for t in range(6):
            sel = rng.choice(len(x), len(x) // 10, replace=False)
            ux = np.clip(x[sel] + rng.normal(0, 20.0, len(sel)), 0, 22500)
            uy = np.clip(y[sel] + rng.normal(0, 20.0, len(sel)), 0, 22500)
            x[sel], y[sel] = ux, uy
            g.update(T(snap.ids[sel]), T(ux), T(uy))
            out = g.query_device(*qd, out=out)
            torch.cuda.synchronize()
            want = ref.process_tick(snap.ids, x, y, qi, snap.x[qi], snap.y[qi])
            nres = out["n_results"]
            assert np.array_equal(out["neighbour_ids"][:nres].cpu().numpy(), want.neighbour_ids), t
            assert out["distances"][:nres].cpu().numpy().tobytes() == want.distances.tobytes(), t
            for key in keys:
                assert getattr(g.last_metrics, key) == getattr(ref.last_metrics, key), (t, key)
        cap, rep = g.graph_stats
        assert rep >= 3, (cap, rep)


def test_onepass_partition_overflow_redo():
    """Steady-state ticks partition the store in one pass over bucket regions
    planned from the previous tick's counts; when the objects pile into a few
    leaves without a rebuild, a bucket outgrows its region and the tick is
    redone with the two-pass partition -- every tick still equals the oracle."""
    rng = np.random.default_rng(21)
    n, k = 60_000, 16
    snap = synth.place(n, "uniform", seed=8)
    x, y = snap.x.copy(), snap.y.copy()
    with Engine(EngineConfig(k=k, region=synth.REGION, rebuild_window=50)) as eng:
        for t in range(5):
            if t == 2:  # 80 % of the objects jump into one small square
                sel = rng.random(n) < 0.8
                x[sel] = rng.uniform(1000.0, 1300.0, sel.sum())
                y[sel] = rng.uniform(2000.0, 2300.0, sel.sum())
            elif t > 0:
                x = np.clip(x + rng.normal(0, 5.0, n), 0, 22500)
                y = np.clip(y + rng.normal(0, 5.0, n), 0, 22500)
            qsel = rng.choice(n, 3000, replace=False)
            qi, qx, qy = snap.ids[qsel], x[qsel], y[qsel]
            res = eng.process_tick(snap.ids, x, y, qi, qx, qy)
            assert eng.last_metrics.rebuild_flag == (1 if t == 0 else 0)
            assert_same(res, orc.brute_force_knn(snap.ids, x, y, qi, qx, qy, k))


def test_device_calls_follow_the_torch_stream():
    """Tensors produced on a side stream (async pinned copies, a sleep kernel
    ahead of them) feed update/query_device/tick_device on that stream: the
    engine follows torch's current stream, so it never reads them early."""
    snap = synth.place(40_000, "gaussian", seed=6, hotspots=4)
    qi, qx, qy = synth.queries(snap, 4000, seed=6)
    ups = synth.updates(snap, 0.1, 1, seed=6)
    side = torch.cuda.Stream()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731

    def dev(a):
        torch.cuda._sleep(2_000_000)  # keep the stream busy ahead of the copy
        return pin(a).to("cuda", non_blocking=True)

    want0 = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi, qx, qy, 12)
    after = synth.Snapshot(snap.ids.copy(), snap.x.copy(), snap.y.copy())
    synth.apply_updates(after, *ups)
    want1 = orc.brute_force_knn(after.ids, after.x, after.y, qi, qx, qy, 12)
    with Engine(EngineConfig(k=12, region=synth.REGION)) as eng, torch.cuda.stream(side):
        d = [dev(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
        out = eng.tick_device(*d)
        n = out["n_results"]
        got = out["neighbour_ids"][:n].cpu().numpy()
        assert np.array_equal(got, want0.neighbour_ids)
        eng.update(*[dev(a) for a in (snap.ids, snap.x, snap.y)])
        eng.update(*[dev(a) for a in ups])
        out = eng.query_device(*[dev(a) for a in (qi, qx, qy)])
        n = out["n_results"]
        assert np.array_equal(out["neighbour_ids"][:n].cpu().numpy(), want1.neighbour_ids)
        assert out["distances"][:n].cpu().numpy().tobytes() == want1.distances.tobytes()


def test_audit_pruning_finds_no_violations():
    snap = synth.place(20_000, "gaussian", seed=4, hotspots=5)
    qi, qx, qy = synth.queries(snap, 2000, seed=4)
    with Engine(EngineConfig(k=8, region=synth.REGION, th_quad=64, audit_pruning=True)) as eng:
        eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
    assert m.pruned_leaves > 0 and m.pruning_violations == 0


def test_self_check_rejects_duplicate_ids():
    with Engine(EngineConfig(k=1, region=Rect.square(10.0), th_quad=4, self_check=True)) as eng:
        with pytest.raises(ValueError):
            eng.process_tick(np.array([1, 1]), np.array([1.0, 2.0]), np.array([1.0, 2.0]),
                             np.array([1]), np.array([1.0]), np.array([1.0]))


def test_large_k_unsupported_is_loud():
    with pytest.raises(NotImplementedError):
        with Engine(EngineConfig(k=600, region=Rect.square(10.0))) as eng:
            eng.process_tick(np.arange(3), np.ones(3), np.ones(3), [], [], [])


@pytest.mark.parametrize("dist,n,nq,k,seed", [
    ("gaussian", 1_000_000, 100_000, 32, 3),
    ("uniform", 1_000_000, 100_000, 32, 0),
])
def test_large_vs_oracle_engine_port(dist, n, nq, k, seed):
    """Full-size-class check: every query vs the pinned C port of the
    reference engine (which is itself checked against the reference)."""
    snap = synth.place(n, dist, seed=seed)
    qi, qx, qy = synth.queries(snap, nq, seed=seed)
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, k, synth.REGION, 384)
    assert_same(res, want)
    assert m.distance_evals == want.metrics["distance_evals"]
    assert m.pruned_leaves == want.metrics["pruned_leaves"]
    assert m.active_left == want.metrics["active_left"]
    assert m.active_right == want.metrics["active_right"]


def test_issuer_range_growth_between_ticks():
    """The issuer-order sort is planned from the previous tick's issuer-id
    range; a tick whose range needs more bits must still come out in issuer
    order (the engine re-runs it with the measured range)."""
    rng = np.random.default_rng(21)
    n = 3000
    x = rng.uniform(0, 500, n)
    y = rng.uniform(0, 500, n)
    ids = np.arange(n, dtype=np.int64)
    region = Rect.square(500.0)
    with Engine(EngineConfig(k=9, region=region, th_quad=32)) as eng:
        for t, span in enumerate([40, 40, 1 << 40, 3, 1 << 62]):
            nq = 200
            sel = rng.choice(n, nq, replace=False)
            qx, qy = x[sel], y[sel]
            qi = (rng.integers(0, span, nq) if span > 1 else np.zeros(nq, np.int64)).astype(np.int64)
            qi[: nq // 2] = ids[sel[: nq // 2]]
            res = eng.process_tick(ids, x, y, qi, qx, qy)
            assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, 9))
            assert eng.last_metrics.tick == t


@pytest.mark.parametrize("lo,width", [(0.0, 22500.0), (-7.3, 1000.1), (1e6 + 0.1, 3.0)])
def test_cell_borders_match_reference_encoding(lo, width):
    """Objects exactly on (and one ulp either side of) quadrant borders at
    every level: the device's reciprocal fast path must floor exactly like
    the reference's IEEE division (geometry.py:105-129), so the index and the
    per-leaf cell ranges equal the oracle's build_index / index_objects."""
    rng = np.random.default_rng(int(width))
    region = Rect(lo, lo, lo + width, lo + width)
    pts = []
    for lvl in (1, 3, 5, 8, 10, 13, 16):
        c = rng.integers(0, 2 ** lvl, 300)
        b = lo + np.ldexp(c.astype(np.float64), -lvl) * width
        for v in (b, np.nextafter(b, -np.inf), np.nextafter(b, np.inf)):
            pts.append(v)
    xs = np.concatenate(pts)
    ys = rng.permutation(xs)
    xs = np.concatenate([xs, [lo, lo + width, lo - 1.0, lo + width + 1.0]])
    ys = np.concatenate([ys, [lo + width, lo, lo + 0.5 * width, lo - 3.0]])
    n = len(xs)
    ids = np.arange(n, dtype=np.int64)
    th, l_max = 8, 10
    want_ix = orc.build_index(xs, ys, region, th, l_max)
    want_st = orc.index_objects(ids, xs, ys, region, want_ix)
    orc.free_index(want_ix)
    sel = rng.choice(n, 400, replace=False)
    with Engine(EngineConfig(k=6, region=region, th_quad=th, l_max=l_max)) as eng:
        res = eng.process_tick(ids, xs, ys, ids[sel], xs[sel], ys[sel])
        ix = eng.index
        for key in ("leaf_level", "leaf_code", "leaf_key", "leaf_span", "build_counts"):
            np.testing.assert_array_equal(getattr(ix, key), want_ix[key], err_msg=key)
        cs, ce = eng.cell_ranges()
        np.testing.assert_array_equal(cs, want_st["cell_start"])
        np.testing.assert_array_equal(ce, want_st["cell_end"])
        assert eng.last_metrics.clamped_objects == want_st["clamped"]
    assert_same(res, orc.brute_force_knn(ids, xs, ys, ids[sel], xs[sel], ys[sel], 6))


@pytest.mark.parametrize("n,k", [(5000, 16), (20, 32)])
def test_pinned_host_outputs_written_in_place(n, k):
    """Pinned (device-mapped) host output buffers are written by the search
    kernel directly; full rows and short rows (n - 1 < k) both match."""
    rng = np.random.default_rng(n)
    x = rng.uniform(0, 100, n)
    y = rng.uniform(0, 100, n)
    ids = np.arange(n, dtype=np.int64) * 3
    nq = min(n, 700)
    sel = rng.choice(n, nq, replace=False)
    qi, qx, qy = ids[sel], x[sel], y[sel]
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
    out = (pin(nq, torch.int64), pin(nq, torch.int32), pin(nq * k, torch.int64),
           pin(nq * k, torch.float64))
    offs = np.full(nq + 1, -7, np.int64)
    want = orc.brute_force_knn(ids, x, y, qi, qx, qy, k)
    with Engine(EngineConfig(k=k, region=Rect.square(100.0), th_quad=24)) as eng:
        for _ in range(2):
            res = eng.process_tick(ids, x, y, qi, qx, qy, out=out)
            assert_same(res, want)
            # optional caller-owned offsets buffer: filled in place
            res = eng.process_tick(ids, x, y, qi, qx, qy, out=out + (offs,))
            assert_same(res, want)
            assert res.offsets is offs and np.array_equal(offs, want.offsets)


def test_sliced_host_tick_equals_device_tick():
    """Host ticks of >= 64K queries search in result-row slices whose copies
    overlap the next slice; the CSR must equal the device-resident tick's and
    a brute-force sample."""
    snap = synth.place(200_000, "gaussian", seed=8, hotspots=6, sigma=900.0)
    qi, qx, qy = synth.queries(snap, 90_000, seed=8)
    with Engine(EngineConfig(k=12, region=synth.REGION)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
        out = eng.tick_device(T(snap.ids), T(snap.x), T(snap.y), T(qi), T(qx), T(qy))
        nres = out["n_results"]
        np.testing.assert_array_equal(res.query_ids, out["query_ids"][:len(qi)].cpu().numpy())
        np.testing.assert_array_equal(res.neighbour_ids, out["neighbour_ids"][:nres].cpu().numpy())
        assert res.distances.tobytes() == out["distances"][:nres].cpu().numpy().tobytes()
    rows = np.sort(np.random.default_rng(0).choice(len(qi), 300, replace=False))
    order = np.argsort(qi, kind="stable")
    want = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi[order[rows]], qx[order[rows]],
                               qy[order[rows]], 12)
    for j, r in enumerate(rows):
        a, b = res.offsets[r], res.offsets[r + 1]
        np.testing.assert_array_equal(res.neighbour_ids[a:b],
                                      want.neighbour_ids[want.offsets[j]:want.offsets[j + 1]])


def test_sliced_host_tick_short_rows():
    """Sliced host tick whose rows are short (fewer objects than k): the
    compacted CSR replaces the row copies."""
    rng = np.random.default_rng(3)
    n, nq, k = 20, 70_000, 32
    x = rng.uniform(0, 10, n)
    y = rng.uniform(0, 10, n)
    ids = np.arange(n, dtype=np.int64)
    qi = rng.integers(0, 40, nq).astype(np.int64)  # issuers in and out of the snapshot
    qx = rng.uniform(0, 10, nq)
    qy = rng.uniform(0, 10, nq)
    with Engine(EngineConfig(k=k, region=Rect.square(10.0), th_quad=4)) as eng:
        res = eng.process_tick(ids, x, y, qi, qx, qy)
    assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, k))


@pytest.mark.parametrize("k,th", [(32, 16), (32, 128), (64, 64), (128, 256)])
def test_near_ties_at_the_cut(k, th):
    """A jittered lattice: many candidate distances agree to ~1e-9 relative,
    so the 32/64-bit key networks see equal truncated keys everywhere --
    including across the cut between kept and dropped candidates, where the
    exact (d2, id) network must decide (regression: a missed neighbour
    0.7 ppm closer than the kept 32nd)."""
    rng = np.random.default_rng(k + th)
    g = np.arange(48, dtype=np.float64)
    gx, gy = np.meshgrid(g, g)
    x = gx.ravel() + rng.uniform(-1e-7, 1e-7, gx.size) + 1.0
    y = gy.ravel() + rng.uniform(-1e-7, 1e-7, gy.size) + 1.0
    n = len(x)
    ids = rng.permutation(n).astype(np.int64)
    sel = rng.choice(n, 800, replace=False)
    qi, qx, qy = ids[sel], x[sel] + rng.uniform(-1e-8, 1e-8, 800), y[sel]
    with Engine(EngineConfig(k=k, region=Rect.square(50.0), th_quad=th)) as eng:
        res = eng.process_tick(ids, x, y, qi, qx, qy)
    assert_same(res, orc.brute_force_knn(ids, x, y, qi, qx, qy, k))


def test_cfg3_full_size_vs_engine_port():
    """BASELINE.json configs[2] at full size (Gaussian/16, 10M objects, 1M
    queries, k=32): every row and the per-tick metrics against the pinned C
    port of the reference engine (OpenMP on the host cores)."""
    snap = synth.place(10_000_000, "gaussian", seed=3)
    qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
    with Engine(EngineConfig(k=32, region=synth.REGION)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, 32, synth.REGION, 384)
    assert_same(res, want)
    assert m.distance_evals == want.metrics["distance_evals"]
    assert m.pruned_leaves == want.metrics["pruned_leaves"]
    assert m.active_left == want.metrics["active_left"]
    assert m.active_right == want.metrics["active_right"]


def test_cfg4_full_size_vs_engine_port():
    """BASELINE.json configs[3] on one GPU (uniform, 100M objects, 10M
    queries, k=16): every row and the metrics against the C engine port."""
    snap = synth.place(100_000_000, "uniform", seed=4)
    qi, qx, qy = synth.queries(snap, 10_000_000, seed=4)
    with Engine(EngineConfig(k=16, region=synth.REGION)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, 16, synth.REGION, 192)
    assert_same(res, want)
    assert m.distance_evals == want.metrics["distance_evals"]
    assert m.pruned_leaves == want.metrics["pruned_leaves"]


@pytest.mark.parametrize("dist", ["uniform", "gaussian", "coincident"])
def test_incremental_store_matches_full_rebuild(dist):
    """Delta ticks re-index incrementally (only the moved slots change key):
    over many ticks -- repeated updates of an id between queries, updates
    in several batches, new ids appended, moves out of / back into the
    region, a query with no update -- every result and metric (incl.
    clamped_objects) equals a full-snapshot tick on the carried-forward
    snapshot.  "coincident": 40 % of the objects sit on 20 shared points and
    updates move objects onto / off them, so old key groups far longer than
    the scanned limit take the slot -> position map path (k_moved_deferred)."""
    rng = np.random.default_rng(7)
    n = 40_000
    spots = None
    if dist == "coincident":
        snap = synth.place(n, "uniform", seed=12)
        spots = rng.uniform(0, 22500, (20, 2))
        on = rng.random(n) < 0.4
        pick = rng.integers(0, 20, n)
        snap.x[on], snap.y[on] = spots[pick[on], 0], spots[pick[on], 1]
    else:
        snap = synth.place(n, dist, seed=12, hotspots=5, sigma=700.0)
    ids = list(snap.ids)
    xs, ys = list(snap.x), list(snap.y)
    pos = {int(i): j for j, i in enumerate(snap.ids)}
    with Engine(EngineConfig(k=16, region=synth.REGION)) as full, \
            Engine(EngineConfig(k=16, region=synth.REGION)) as delta:
        delta.load(snap.ids, snap.x, snap.y)
        for t in range(8):
            for _ in range(int(rng.integers(0, 3))):  # 0-2 update batches before the query
                u = int(rng.integers(50, 3000))
                uid = rng.choice(np.asarray(ids), u, replace=True)  # repeats inside a batch
                ux = rng.uniform(-800, 23300, u)  # some outside the region [0, 22500]
                uy = rng.uniform(-800, 23300, u)
                if spots is not None:  # half of the moves land on a shared point
                    on = rng.random(u) < 0.5
                    pick = rng.integers(0, 20, u)
                    ux[on], uy[on] = spots[pick[on], 0], spots[pick[on], 1]
                if rng.random() < 0.5:  # brand-new ids
                    new = np.arange(10 ** 9 + len(ids), 10 ** 9 + len(ids) + 7)
                    uid = np.concatenate([uid, new])
                    ux = np.concatenate([ux, rng.uniform(0, 22500, 7)])
                    uy = np.concatenate([uy, rng.uniform(0, 22500, 7)])
                delta.update(uid, ux, uy)
                for i, x, y in zip(uid, ux, uy):  # carry forward, last update wins
                    i = int(i)
                    if i not in pos:
                        pos[i] = len(ids)
                        ids.append(i)
                        xs.append(x)
                        ys.append(y)
                    else:
                        xs[pos[i]], ys[pos[i]] = x, y
            A, X, Y = np.asarray(ids, np.int64), np.asarray(xs), np.asarray(ys)
            sel = rng.choice(len(A), 2000, replace=False)
            qi, qx, qy = A[sel], X[sel], Y[sel]
            a = full.process_tick(A, X, Y, qi, qx, qy)
            b = delta.query(qi, qx, qy)
            assert_same(b, a)
            for key in ("distance_evals", "pruned_leaves", "clamped_objects", "rebuild_flag",
                        "active_left", "active_right"):
                assert getattr(delta.last_metrics, key) == getattr(full.last_metrics, key), (t, key)
        assert delta.snapshot_size == len(ids)


def test_self_check_validates_every_rebuilt_index(monkeypatch):
    """engine.py:620-621: with self_check the rebuilt index is validated
    (quadindex.py:51-76) -- on the first tick and on a should_rebuild tick;
    a corrupted export is rejected with AssertionError."""
    from paper_1412_6170_b200 import index as ix_mod

    calls = []
    real = ix_mod.QuadIndex.validate
    monkeypatch.setattr(ix_mod.QuadIndex, "validate",
                        lambda self, *a, **kw: (calls.append(self.n_leaves), real(self, *a, **kw)))
    snap = synth.place(60_000, "uniform", seed=9)
    with Engine(EngineConfig(k=8, region=synth.REGION, self_check=True, rebuild_window=1,
                             rebuild_factor=1.2)) as eng:
        for t in range(3):
            if t == 2:  # a cluster: evaluations jump, the next tick rebuilds
                snap.x[: 30_000] = 5000.0 + snap.x[: 30_000] * 1e-3
                snap.y[: 30_000] = 9000.0 + snap.y[: 30_000] * 1e-3
            qi, qx, qy = synth.queries(snap, 2000, seed=t)
            eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        qi, qx, qy = synth.queries(snap, 2000, seed=7)
        eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        assert eng.last_metrics.rebuild_flag == 1
        assert len(calls) == 2
        bad = eng.index
        bad.leaf_span[0] += 1
        with pytest.raises(AssertionError):
            real(bad)


def test_two_engines_large_k_in_one_process():
    """k > 32 kernels need a >48 KB shared-memory attribute, which is per
    device: two engines (every visible device, or the same one twice) in
    one process both run."""
    n_dev = torch.cuda.device_count()
    devs = [0, 1] if n_dev > 1 else [0, 0]
    snap = synth.place(20_000, "gaussian", seed=10, hotspots=3)
    qi, qx, qy = synth.queries(snap, 1500, seed=10)
    want = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi, qx, qy, 128)
    engines = [Engine(EngineConfig(k=128, region=synth.REGION, device=d)) for d in devs]
    try:
        for eng in engines:
            assert_same(eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy), want)
    finally:
        for eng in engines:
            eng.close()


def test_repeated_issuers_on_a_wider_id_range():
    """Advisor finding: repeated issuer ids on a tick whose id range needs
    more bits than the previous tick's (the bitmap planned from the old
    range sees ids beyond it): the tick still comes out in stable issuer
    order, and a later tick with a narrower range as well."""
    rng = np.random.default_rng(31)
    n = 4000
    x = rng.uniform(0, 300, n)
    y = rng.uniform(0, 300, n)
    ids = np.arange(n, dtype=np.int64)
    region = Rect.square(300.0)
    with Engine(EngineConfig(k=5, region=region, th_quad=24)) as eng:
        for t, (span, nq) in enumerate([(64, 60), (1 << 30, 900), (1 << 33, 80), (50, 300)]):
            sel = rng.choice(n, nq, replace=False)
            qi = rng.integers(0, span, nq).astype(np.int64)
            qi[nq // 3: nq // 3 + 5] = qi[0]  # repeats
            res = eng.process_tick(ids, x, y, qi, x[sel], y[sel])
            assert_same(res, orc.brute_force_knn(ids, x, y, qi, x[sel], y[sel], 5))
            assert eng.last_metrics.tick == t


@pytest.mark.parametrize("k", [100, 200, 512])
def test_grouped_navigation_metrics_vs_port(k):
    """k > 64 runs each query's navigate calls on a lane group (navigate_grp:
    the levels of the descent chain evaluated at once).  Rows, prune events,
    iterations and active counts equal the reference engine's serial walk
    (engine.py:396-503), and the prune audit (engine.py:529-554) runs through
    the grouped path without violations."""
    from paper_1412_6170_b200.engine import resolve_th_quad
    snap = synth.place(60_000, "gaussian", seed=21, hotspots=5, sigma=700.0)
    qi, qx, qy = synth.queries(snap, 3000, seed=21)
    th = resolve_th_quad("auto", k)
    with Engine(EngineConfig(k=k, region=synth.REGION, audit_pruning=True)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, k, synth.REGION, th)
    assert_same(res, want)
    for key in ("distance_evals", "pruned_leaves", "iterations_left", "iterations_right",
                "active_left", "active_right"):
        assert getattr(m, key) == want.metrics[key], (key, getattr(m, key), want.metrics[key])
    assert m.pruned_leaves > 0 and m.pruning_violations == 0


@pytest.mark.parametrize("k", [8, 32, 128])
def test_phase_split_first_iteration(k):
    """engine.py:641-642 reports first_iteration and the direction loop as two
    phases; the device runs both in one kernel per query batch and splits the
    kernel's event time by the batches' measured own-leaf warp time."""
    snap = synth.place(200_000, "uniform", seed=5)
    qi, qx, qy = synth.queries(snap, 50_000, seed=5)
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        for _ in range(2):
            eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
            m = eng.last_metrics
            assert m.t_first_iteration_us > 0 and m.t_loop_us >= 0
            assert m.t_first_iteration_us + m.t_loop_us < m.t_total_us


class _DLPackOnly:
    """A device array seen only through the DLPack protocol (as CuPy / JAX
    arrays are)."""

    def __init__(self, t):
        self._t = t

    def __dlpack__(self, *args, **kw):
        return self._t.__dlpack__(*args, **kw)

    def __dlpack_device__(self):
        return self._t.__dlpack_device__()


def test_device_paths_take_and_give_dlpack():
    """device-resident inputs and results through DLPack --
    any DLPack producer is taken zero-copy, the results are DLPack producers,
    and a wrong dtype fails loudly instead of being read as raw bytes."""
    snap = synth.place(30_000, "uniform", seed=8)
    qi, qx, qy = synth.queries(snap, 3_000, seed=8)
    d = [torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")
         for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
    with Engine(EngineConfig(k=16, region=synth.REGION)) as eng:
        want = {k: v.clone() if hasattr(v, "clone") else v for k, v in eng.tick_device(*d).items()}
        got = eng.tick_device(*[_DLPackOnly(t) for t in d])
        for key in ("query_ids", "lengths", "offsets", "neighbour_ids", "distances"):
            view = torch.from_dlpack(got[key].__dlpack__())
            assert view.data_ptr() == got[key].data_ptr()
            assert torch.equal(view, want[key]), key
        eng.load(snap.ids, snap.x, snap.y)
        upd = synth.updates(snap, 0.1, 0, seed=8)
        eng.update(*[_DLPackOnly(torch.as_tensor(np.ascontiguousarray(a), device="cuda:0"))
                     for a in upd])
        q = eng.query_device(*[_DLPackOnly(t) for t in d[3:]])
        assert q["n_results"] == 3_000 * 16
        with pytest.raises(TypeError):
            eng.tick_device(d[0].to(torch.int32), *d[1:])
