"""Every BASELINE.json configuration as BASELINE defines it, at full size,
against the pinned C port of the reference engine and the brute-force
certificate:

* configs[1] (cfg2): uniform 1M objects, 100K queries per tick, k=32, a
  snapshot at tick 0 then 9 ticks of 10 % position updates through the delta
  API (load / update / query, datasets.py:136-148 carry-forward) -- every
  tick's rows, metrics and rebuild flag against ``engine_tick`` on the
  carried-forward snapshot with the index positions of the last rebuild;
* a >= 1M-object sequence whose ``should_rebuild`` (quadindex.py:231-246)
  fires mid-run, through both the full-snapshot and the delta API;
* configs[4] (cfg5): k = 8 and k = 128 on the 10M Gaussian objects with the
  full 1M queries;
* configs[2] stress variant: Gaussian hotspots=1.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1412_6170_b200 import Engine, EngineConfig, synth
from paper_1412_6170_b200.engine import resolve_th_quad
from paper_1412_6170_b200.verify import certify

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = torch.device("cuda", 0)
METRIC_KEYS = ("distance_evals", "pruned_leaves", "iterations_left", "iterations_right",
               "active_left", "active_right", "clamped_objects")


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def _should_rebuild(history, window=3, factor=1.5):
    """quadindex.py:231-246, restated for the test's own bookkeeping."""
    if len(history) < window + 1:
        return False
    return history[-1] > factor * (sum(history[-window - 1:-1]) / window)


def _assert_same(res, want):
    np.testing.assert_array_equal(res.query_ids, want.query_ids)
    np.testing.assert_array_equal(res.lengths, want.lengths)
    np.testing.assert_array_equal(res.neighbour_ids, want.neighbour_ids)
    assert res.distances.tobytes() == want.distances.tobytes()


def _assert_metrics(m, want, tag):
    for key in METRIC_KEYS:
        assert getattr(m, key) == want[key], (tag, key, getattr(m, key), want[key])


def _certify_host(snap, qi, qx, qy, k, res):
    """The brute-force certificate of a host TickResult (all (query, object)
    pairs on the device)."""
    nq = len(qi)
    out = dict(query_ids=_t(res.query_ids), lengths=_t(res.lengths), offsets=_t(res.offsets),
               neighbour_ids=_t(res.neighbour_ids), distances=_t(res.distances),
               n_results=len(res.neighbour_ids))
    bad = certify(_t(snap.ids), _t(snap.x), _t(snap.y), _t(qi), _t(qx), _t(qy), k, out)
    assert all(v == 0 for v in bad.values()), bad
    assert nq == len(res.query_ids)


class _PortTicks:
    """The reference engine's tick sequence (engine.py:601-696) through the
    C port: the index is rebuilt from the positions of the tick on which
    should_rebuild (or the first tick) fires, and reused otherwise."""

    def __init__(self, k):
        self.k = k
        self.th = resolve_th_quad("auto", k)
        self.history = []
        self.build_xy = None

    def tick(self, snap, qi, qx, qy):
        rebuild = self.build_xy is None or _should_rebuild(self.history)
        if rebuild:
            self.build_xy = (snap.x.copy(), snap.y.copy())
        want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, self.k, synth.REGION,
                               self.th, build_xy=self.build_xy)
        self.history.append(want.metrics["distance_evals"])
        return want, int(rebuild)


def test_cfg2_delta_sequence_vs_port_and_certificate():
    """BASELINE.json configs[1]: uniform 1M, 100K queries per tick, k=32,
    tick 0 = load + query, then 9 ticks of 10 % updates + query."""
    k = 32
    snap = synth.place(1_000_000, "uniform", seed=0)
    port = _PortTicks(k)
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        eng.load(snap.ids, snap.x, snap.y)
        for t in range(10):
            if t:
                uid, ux, uy = synth.updates(snap, 0.10, t, seed=0)
                eng.update(uid, ux, uy)
                synth.apply_updates(snap, uid, ux, uy)
            qi, qx, qy = synth.queries(snap, 100_000, seed=1000 + t)
            res = eng.query(qi, qx, qy)
            want, rebuild = port.tick(snap, qi, qx, qy)
            _assert_same(res, want)
            _assert_metrics(eng.last_metrics, want.metrics, t)
            assert eng.last_metrics.rebuild_flag == rebuild, t
            assert eng.last_metrics.n_objects == 1_000_000
            if t in (0, 9):
                _certify_host(snap, qi, qx, qy, k, res)


def _collapse(snap, frac, t, seed):
    """Move a fraction of the objects into one Gaussian cluster (the index
    built on the spread-out positions then holds huge own leaves, so the
    distance evaluations jump and should_rebuild fires next tick)."""
    rng = np.random.default_rng([seed, t])
    n = len(snap.ids)
    sel = rng.choice(n, int(n * frac), replace=False)
    ux = np.clip(rng.normal(7000.0, 300.0, sel.size), 0.0, 22500.0)
    uy = np.clip(rng.normal(15000.0, 300.0, sel.size), 0.0, 22500.0)
    return snap.ids[sel].copy(), ux, uy


@pytest.mark.parametrize("api", ["snapshot", "delta"])
def test_rebuild_fires_mid_sequence_1m(api):
    """A 1M-object sequence: four quiet ticks, then 40 % of the objects move
    into one cluster; the reference's should_rebuild fires on the following
    tick.  Every tick's rows, metrics and rebuild flag equal the port's."""
    k = 16
    snap = synth.place(1_000_000, "uniform", seed=21)
    port = _PortTicks(k)
    flags = []
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        if api == "delta":
            eng.load(snap.ids, snap.x, snap.y)
        for t in range(8):
            if t == 4:
                upd = _collapse(snap, 0.4, t, seed=21)
            elif t:
                upd = synth.updates(snap, 0.05, t, seed=21)
            if t:
                if api == "delta":
                    eng.update(*upd)
                synth.apply_updates(snap, *upd)
            qi, qx, qy = synth.queries(snap, 100_000, seed=2000 + t)
            if api == "delta":
                res = eng.query(qi, qx, qy)
            else:
                res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
            want, rebuild = port.tick(snap, qi, qx, qy)
            _assert_same(res, want)
            _assert_metrics(eng.last_metrics, want.metrics, t)
            assert eng.last_metrics.rebuild_flag == rebuild, t
            flags.append(rebuild)
    assert flags[0] == 1 and sum(flags[1:5]) == 0 and 1 in flags[5:], flags


@pytest.mark.parametrize("k", [8, 128])
def test_cfg5_k_sweep_full_size(k):
    """BASELINE.json configs[4] at full size: the 10M Gaussian/16 objects and
    all 1M queries, every row and metric against the port, and every row
    certified by brute force."""
    snap = synth.place(10_000_000, "gaussian", seed=3)
    qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
    d = [_t(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        out = eng.tick_device(*d)
        torch.cuda.synchronize()
        m = eng.last_metrics
        bad = certify(*d, k, out)
        assert all(v == 0 for v in bad.values()), bad
        nres = out["n_results"]
        got_ids = out["neighbour_ids"][:nres].cpu().numpy()
        got_d = out["distances"][:nres].cpu().numpy()
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, k, synth.REGION,
                           resolve_th_quad("auto", k))
    np.testing.assert_array_equal(got_ids, want.neighbour_ids)
    assert got_d.tobytes() == want.distances.tobytes()
    _assert_metrics(m, want.metrics, k)


def test_cfg3_single_hotspot_stress():
    """SURVEY §8(d) cfg3 stress variant: Gaussian with hotspots=1 (thousands
    of overfull leaves), 10M objects, 1M queries, k=32."""
    snap = synth.place(10_000_000, "gaussian", seed=3, hotspots=1)
    qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
    with Engine(EngineConfig(k=32, region=synth.REGION)) as eng:
        res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        m = eng.last_metrics
        assert eng.index.overfull_leaves > 1000
    want = orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, 32, synth.REGION, 384)
    _assert_same(res, want)
    _assert_metrics(m, want.metrics, "hotspots=1")
    _certify_host(snap, qi, qx, qy, 32, res)
