"""Result consumers of the tick boundary.

``write_result_block`` mirrors reference pkg/src/mknn/studies.py:105-108
(same signature, same bytes): one CSV line per neighbour,
``f"{tick},{query_id},{rank},{neighbour_id},{distance:.9g}\\n"``, in row
order.  The lines are formatted by the native library on all host threads
(``mknn_format_result_rows``) instead of a Python loop over every neighbour.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N

RESULT_HEADER = "tick,query_id,rank,neighbour_id,distance"  # studies.py:102


def format_result_rows(tick: int, result, threads: int = 0) -> bytes:
    """The CSV lines of one TickResult (studies.py:105-108), as bytes."""
    qids = np.ascontiguousarray(result.query_ids, dtype=np.int64)
    offsets = np.ascontiguousarray(result.offsets, dtype=np.int64)
    nids = np.ascontiguousarray(result.neighbour_ids, dtype=np.int64)
    dist = np.ascontiguousarray(result.distances, dtype=np.float64)
    nq = len(qids)
    if nq == 0:
        return b""
    cap = 100 * int(offsets[-1] - offsets[0]) + 1
    buf = np.empty(cap, np.uint8)  # not zero-filled
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    n = N.lib().mknn_format_result_rows(int(tick), nq, p(qids), p(offsets), p(nids), p(dist),
                                        p(buf), cap, int(threads))
    if n < 0:
        raise RuntimeError(f"mknn_format_result_rows failed ({n})")
    return buf[:n].tobytes()


def write_result_block(f, tick: int, result) -> None:
    """studies.py:105-108: append the tick's rows to the text file ``f``."""
    f.write(format_result_rows(tick, result).decode("ascii"))
