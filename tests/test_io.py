"""Native result formatter vs the reference's write_result_block
(studies.py:105-108, restated here as its f-string loop).  Host-only."""

import io

import numpy as np

from paper_1412_6170_b200.engine import TickResult
from paper_1412_6170_b200.io import RESULT_HEADER, format_result_rows, write_result_block


def reference_block(tick, res) -> str:
    out = []
    for qid, ids, dists in res.iter_rows():  # studies.py:106-108
        for r in range(len(ids)):
            out.append(f"{tick},{qid},{r},{ids[r]},{dists[r]:.9g}\n")
    return "".join(out)


def make_result(rng, nq, k):
    lens = rng.integers(0, k + 1, nq).astype(np.int32)
    offsets = np.zeros(nq + 1, np.int64)
    np.cumsum(lens, out=offsets[1:])
    m = int(offsets[-1])
    d = np.abs(rng.standard_normal(m)) * 10.0 ** rng.integers(-8, 9, m)
    if m > 5:
        d[:5] = [0.0, np.inf, 1e-310, 123456789.5, 2.0 ** -1074]
    return TickResult(query_ids=np.sort(rng.integers(-10**12, 10**12, nq)), lengths=lens,
                      offsets=offsets, neighbour_ids=rng.integers(-2**62, 2**62, m),
                      distances=d)


def test_format_matches_reference_loop():
    rng = np.random.default_rng(0)
    for nq, k in ((0, 4), (1, 1), (7, 3), (5000, 32)):
        res = make_result(rng, nq, k)
        for tick in (0, 17, -3):
            assert format_result_rows(tick, res).decode() == reference_block(tick, res)
            assert format_result_rows(tick, res, threads=1).decode() == reference_block(tick, res)


def test_write_result_block_appends():
    res = make_result(np.random.default_rng(1), 100, 8)
    f = io.StringIO()
    f.write(RESULT_HEADER + "\n")
    write_result_block(f, 3, res)
    assert f.getvalue() == RESULT_HEADER + "\n" + reference_block(3, res)
