"""Host-side logic of the drop-in boundary (no GPU): config validation, the
th_quad rule, metrics CSV schema, the rebuild rule, QuadIndex invariants.
Mirrors the reference tests test_engine.py:35-41, 367-376 and
test_quadindex.py:224-241 for the same API."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1412_6170_b200 import EngineConfig, QuadIndex, Rect, TickMetrics, resolve_th_quad
from paper_1412_6170_b200 import should_rebuild
from paper_1412_6170_b200.index import encode_points


def test_resolve_th_quad_rule():
    assert resolve_th_quad("auto", 1) == 192
    assert resolve_th_quad("auto", 31) == 192
    assert resolve_th_quad("auto", 32) == 384
    assert resolve_th_quad("auto", 128) == 1536
    assert resolve_th_quad("auto", 129) == 2048
    assert resolve_th_quad(77, 32) == 77


def test_engine_config_validation():
    with pytest.raises(ValueError):
        EngineConfig(k=0, region=Rect.square(10.0))
    with pytest.raises(ValueError):
        EngineConfig(k=1, region=Rect.square(10.0), threads=0)
    with pytest.raises(ValueError):
        EngineConfig(k=1, region=Rect.square(10.0), th_quad="sometimes")
    with pytest.raises(ValueError):
        EngineConfig(k=1, region=Rect.square(10.0), num_bins=1)
    with pytest.raises(ValueError):
        EngineConfig(k=1, region=Rect.square(10.0), rebuild_window=0)
    with pytest.raises(ValueError):
        EngineConfig(k=1, region=Rect.square(10.0), rebuild_factor=0.0)


def test_rect_validation():
    with pytest.raises(ValueError):
        Rect(1.0, 0.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        Rect(0.0, float("nan"), 1.0, 1.0)
    r = Rect.square(22500.0)
    assert r.width == 22500.0 and r.contains(0.0, 22500.0)


def test_metrics_csv_schema():
    m = TickMetrics(tick=3, n_objects=10, n_queries=2)
    assert TickMetrics.csv_header().startswith("tick,n_objects,n_queries")
    assert len(m.csv_row().split(",")) == len(TickMetrics.CSV_FIELDS) == 14


def test_should_rebuild_rule():
    assert should_rebuild([100, 100, 100, 500], window=3, factor=1.5) is True
    assert should_rebuild([100, 100, 100, 150], window=3, factor=1.5) is False
    assert should_rebuild([100, 100, 100, 100], window=3, factor=1.0) is False
    assert should_rebuild([100, 500], window=3, factor=1.5) is False
    assert should_rebuild([], window=3, factor=1.5) is False
    with pytest.raises(ValueError):
        should_rebuild([1, 2], window=0)


def test_host_encode_matches_oracle():
    rng = np.random.default_rng(3)
    region = Rect.square(1024.0)
    x = rng.uniform(-10, 1040, 500)
    y = rng.uniform(-10, 1040, 500)
    for lvl in (0, 3, 10):
        got = encode_points(x, y, region, lvl)
        want = [orc.encode(a, b, region, lvl) for a, b in zip(x, y)]
        assert got.tolist() == want


def _qi_from_oracle(ix, region, th, l_max):
    return QuadIndex(mbr=region, th_quad=th, l_max=l_max, l_deep=ix["l_deep"],
                     leaf_level=ix["leaf_level"], leaf_code=ix["leaf_code"],
                     leaf_key=ix["leaf_key"], leaf_span=ix["leaf_span"], z_map=ix["z_map"],
                     build_counts=ix["build_counts"], n_build=0,
                     overfull_leaves=ix["overfull_leaves"])


def test_quadindex_validate_and_negative_controls():
    """test_acceptance.py:92-141 criterion 3 on the host QuadIndex view."""
    rng = np.random.default_rng(1)
    region = Rect.square(22500.0)
    x = rng.uniform(0, 22500.0, 200)
    y = rng.uniform(0, 22500.0, 200)
    ix = orc.build_index(x, y, region, 16, 4)
    try:
        qi = _qi_from_oracle(ix, region, 16, 4)
        qi.validate()
        for corrupt in ("cover", "capacity", "locate"):
            bad = _qi_from_oracle(ix, region, 16, 4)
            if corrupt == "cover":
                bad.leaf_span = bad.leaf_span.copy()
                bad.leaf_span[0] += 1
            elif corrupt == "capacity":
                j = int(np.argmin(bad.leaf_level))
                bad.build_counts = bad.build_counts.copy()
                bad.build_counts[j] = bad.th_quad + 1
            else:
                bad.z_map = bad.z_map.copy()
                other = int(np.flatnonzero(bad.z_map != bad.z_map[0])[0])
                bad.z_map[0] = bad.z_map[other]
            with pytest.raises(AssertionError):
                bad.validate()
    finally:
        orc.free_index(ix)
