"""Pin the C oracle (oracle/mknn_oracle.c) to the real reference.

Every fixture under tests/golden/ was produced by the reference package
itself (tests/golden/make_golden.py).  These tests run on CPU only.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from tests import golden as G

CASES = G.case_names()

# Fixtures whose reference metrics legitimately differ from the canonical
# port: the reference prunes a quadrant whose min-dist2 EQUALS the k-th d2
# (engine.py:447) and trims boundary ties by scan order (engine.py:220-252),
# the port (and the GPU path) prunes only on a strict excess so the canonical
# lowest-id tie member is always reachable (SURVEY.md §7 hard part 2).
# Distances are identical in every case.
DEGENERATE_TIES = {"hand_collinear_ties", "lattice_shuffled_ids_k8", "lattice_shuffled_ids_k32",
                   "duplicate_coords_k17"}


def _build_xy(case, t):
    """Positions of the tick whose index is in force at tick t
    (engine.py:615-623: rebuild on tick 0 and when should_rebuild fires)."""
    last = 0
    for i in range(t + 1):
        if case.ticks[i].meta["metrics"]["rebuild_flag"]:
            last = i
    return case.ticks[last].x, case.ticks[last].y


def _check_result(res, tick):
    assert G.result_digest(res) == tick.meta["oracle_digest"]
    if tick.has("o_nids"):
        np.testing.assert_array_equal(res.query_ids, tick["o_qids"])
        np.testing.assert_array_equal(res.lengths, tick["o_lens"])
        np.testing.assert_array_equal(res.neighbour_ids, tick["o_nids"])
        assert res.distances.tobytes() == tick["o_dist"].tobytes()


@pytest.mark.parametrize("name", CASES)
def test_brute_force_matches_reference_oracle(name):
    case = G.load(name)
    for tick in case.ticks:
        res = orc.brute_force_knn(tick.ids, tick.x, tick.y, tick.qi, tick.qx, tick.qy, case.k)
        _check_result(res, tick)


@pytest.mark.parametrize("name", CASES)
def test_build_index_matches_reference(name):
    case = G.load(name)
    for t, tick in enumerate(case.ticks):
        bx, by = _build_xy(case, t)
        ix = orc.build_index(bx, by, case.region, G.th_of(case), case.l_max)
        try:
            want = tick.meta["index"]
            assert ix["l_deep"] == want["l_deep"]
            assert ix["n_leaves"] == want["n_leaves"]
            assert ix["overfull_leaves"] == want["overfull_leaves"]
            assert G.digest(ix["z_map"].astype(np.int32)) == want["z_map_digest"]
            st = orc.index_objects(tick.ids, tick.x, tick.y, case.region, ix)
            assert st["clamped"] == want["clamped"]
            if tick.has("ix_leaf_level"):
                for key in ("leaf_level", "leaf_code", "leaf_key", "leaf_span", "build_counts"):
                    np.testing.assert_array_equal(ix[key], tick["ix_" + key], err_msg=key)
                np.testing.assert_array_equal(st["cell_start"], tick["cell_start"])
                np.testing.assert_array_equal(st["cell_end"], tick["cell_end"])
                # stable argsort by l_deep code (quadindex.py:197)
                np.testing.assert_array_equal(st["ids"], tick["store_ids"])
            else:
                assert G.digest(ix["leaf_level"].astype(np.int32), ix["leaf_code"],
                                ix["build_counts"]) == want["leaves_digest"]
                assert G.digest(st["cell_start"], st["cell_end"]) == want["cells_digest"]
        finally:
            orc.free_index(ix)


@pytest.mark.parametrize("name", CASES)
def test_engine_port_matches_reference(name):
    case = G.load(name)
    for t, tick in enumerate(case.ticks):
        res = orc.engine_tick(tick.ids, tick.x, tick.y, tick.qi, tick.qx, tick.qy, case.k,
                              case.region, G.th_of(case), case.l_max, build_xy=_build_xy(case, t))
        _check_result(res, tick)
        want = tick.meta["metrics"]
        m = res.metrics
        assert m["clamped_objects"] == want["clamped_objects"]
        if name in DEGENERATE_TIES:
            continue
        for key in ("distance_evals", "pruned_leaves", "iterations_left", "iterations_right",
                    "active_left", "active_right", "streamed_records"):
            assert m[key] == want[key], (key, m[key], want[key])


def test_cfg1_brute_force_matches_reference():
    """BASELINE.json configs[0]: uniform 100K objects, 10K queries, k=8."""
    from paper_1412_6170_b200 import synth

    meta, arrs = G.load_cfg1()
    snap = synth.place(100_000, "uniform", seed=0)
    assert G.digest(snap.x, snap.y) == meta["input_digest"]  # synth == reference generator
    sel = np.random.default_rng(1).choice(100_000, 10_000, replace=False)
    res = orc.brute_force_knn(snap.ids, snap.x, snap.y, snap.ids[sel], snap.x[sel], snap.y[sel], 8)
    assert G.result_digest(res) == meta["oracle_digest"]
    np.testing.assert_array_equal(res.neighbour_ids, arrs["o_nids"].astype(np.int64))


def test_frozen_geometry_codes():
    from paper_1412_6170_b200.geometry import Rect

    fz = G.load_geometry()
    unit = Rect(0.0, 0.0, 1.0, 1.0)
    for x, y, lvl, code in fz["codes"]:
        assert orc.encode(x, y, unit, lvl) == code
    region = Rect.square(22500.0)
    for lvl in (0, 1, 5, 10, 15):
        got = [orc.encode(x, y, region, lvl) for x, y in zip(fz["enc_px"][:300], fz["enc_py"][:300])]
        assert got == fz[f"enc_l{lvl}"][:300]
