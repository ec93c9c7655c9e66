"""Brute-force certificate: an fp64 device pass over all
(query, object) pairs proves each row is brute_force_knn's (oracle.py:41-106)
at full BASELINE sizes, independently of the engine port.  The checker is
first pinned against the CPU oracle and shown to reject corrupted rows."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1412_6170_b200 import Engine, EngineConfig, synth
from paper_1412_6170_b200.verify import bf_count, certify

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = torch.device("cuda", 0)


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def _tick(snap, qi, qx, qy, k, **cfg):
    d = [_t(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
    eng = Engine(EngineConfig(k=k, region=synth.REGION, **cfg))
    out = eng.tick_device(*d)
    torch.cuda.synchronize()
    return eng, d, out


def _clean(bad):
    assert all(v == 0 for v in bad.values()), bad


def test_bf_count_matches_cpu_count():
    """The device count equals a numpy count of canonical predecessors,
    including exact ties on d2 decided by id, and the issuer skipped."""
    rng = np.random.default_rng(3)
    n, nq = 3000, 700
    x = np.round(rng.uniform(0, 50, n), 1)  # coarse grid: many equal d2
    y = np.round(rng.uniform(0, 50, n), 1)
    ids = rng.permutation(n * 3)[:n].astype(np.int64)
    sel = rng.choice(n, nq, replace=True)
    qi, qx, qy = ids[sel], x[sel], y[sel]
    d2all = (qx[:, None] - x[None, :]) ** 2 + (qy[:, None] - y[None, :]) ** 2
    j = rng.integers(0, n, nq)
    kd = d2all[np.arange(nq), j]
    ki = ids[j]
    want = (((d2all < kd[:, None]) | ((d2all == kd[:, None]) & (ids[None, :] < ki[:, None])))
            & (ids[None, :] != qi[:, None])).sum(1)
    # numpy's (a-b)**2 + (c-d)**2 is the same three roundings as pair_d2
    got = bf_count(_t(ids), _t(x), _t(y), _t(qi), _t(qx), _t(qy), _t(kd), _t(ki)).cpu().numpy()
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("k", [1, 8, 32, 100])
def test_certificate_agrees_with_oracle_and_rejects_corruption(k):
    snap = synth.place(20_000, "gaussian", seed=k, hotspots=3, sigma=600.0)
    qi, qx, qy = synth.queries(snap, 2_000, seed=k)
    eng, d, out = _tick(snap, qi, qx, qy, k)
    with eng:
        want = orc.brute_force_knn(snap.ids, snap.x, snap.y, qi, qx, qy, k)
        n_res = out["n_results"]
        assert np.array_equal(out["neighbour_ids"][:n_res].cpu().numpy(), want.neighbour_ids)
        _clean(certify(*d, k, out))
        # a neighbour replaced by a farther object that is not in the row
        bad = {kk: (v.clone() if hasattr(v, "clone") else v) for kk, v in out.items()}
        r = 5
        o = int(bad["offsets"][r])
        row_ids = set(bad["neighbour_ids"][o:o + k].tolist())
        me = int(out["query_ids"][r])
        far = next(int(i) for i in snap.ids[::-1] if int(i) not in row_ids and int(i) != me)
        bad["neighbour_ids"][o + k - 1] = far
        res = certify(*d, k, bad)
        assert res["distance"] >= 1
        # drop the true last neighbour of a row, keep the list self-consistent
        if k > 1:
            bad = {kk: (v.clone() if hasattr(v, "clone") else v) for kk, v in out.items()}
            bad["lengths"][r] -= 1
            bad["offsets"][r + 1:] -= 1
            keep = torch.ones(n_res, dtype=torch.bool, device=DEV)
            keep[o + k - 1] = False
            bad["neighbour_ids"] = bad["neighbour_ids"][:n_res][keep]
            bad["distances"] = bad["distances"][:n_res][keep]
            bad["n_results"] = n_res - 1
            res = certify(*d, k, bad)
            assert res["count"] == 1 and res["distance"] == 0 and res["order"] == 0


def test_certificate_short_rows_and_tiny_snapshots():
    snap = synth.place(9, "uniform", seed=1)
    qi, qx, qy = synth.queries(snap, 9, seed=1)
    eng, d, out = _tick(snap, qi, qx, qy, 16)
    with eng:
        assert int(out["lengths"][0]) == 8
        _clean(certify(*d, 16, out))


def test_cfg3_full_size_bruteforce_certificate():
    """BASELINE.json configs[2] at full size (Gaussian/16, 10M objects, 1M
    queries, k=32): all 10^13 (query, object) pairs."""
    snap = synth.place(10_000_000, "gaussian", seed=3)
    qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
    eng, d, out = _tick(snap, qi, qx, qy, 32)
    with eng:
        _clean(certify(*d, 32, out))


@pytest.mark.parametrize("k", [1, 128])
def test_k_sweep_bruteforce_certificate(k):
    """BASELINE.json configs[4] ends of the k sweep on the cfg3 objects
    (a 250K-query sample of the 1M, all 10M objects)."""
    snap = synth.place(10_000_000, "gaussian", seed=3)
    qi, qx, qy = synth.queries(snap, 250_000, seed=5)
    eng, d, out = _tick(snap, qi, qx, qy, k)
    with eng:
        _clean(certify(*d, k, out))


def test_cfg4_objects_bruteforce_certificate():
    """BASELINE.json configs[3] objects (uniform 100M, k=16) with a 100K-query
    sample: 10^13 pairs."""
    snap = synth.place(100_000_000, "uniform", seed=4)
    qi, qx, qy = synth.queries(snap, 100_000, seed=4)
    eng, d, out = _tick(snap, qi, qx, qy, 16)
    with eng:
        _clean(certify(*d, 16, out))
