"""Host view of the device quadtree (reference quadindex.py:23-76, 231-246).

``Engine.index`` returns a ``QuadIndex`` copied back from the device on
demand; the arrays have the reference's dtypes and meaning.  ``validate``
re-checks the structural invariants on the host (test / self_check mode
only, never on the hot path).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Rect

MAX_L_MAX = 10  # quadindex.py:20


def _spread(v):
    v = np.asarray(v, dtype=np.int64) & 0xFFFFFFFF
    v = (v | (v << 16)) & 0x0000FFFF0000FFFF
    v = (v | (v << 8)) & 0x00FF00FF00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0F
    v = (v | (v << 2)) & 0x3333333333333333
    v = (v | (v << 1)) & 0x5555555555555555
    return v


def _compact(v):
    v = np.asarray(v, dtype=np.int64) & 0x5555555555555555
    v = (v | (v >> 1)) & 0x3333333333333333
    v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0F
    v = (v | (v >> 4)) & 0x00FF00FF00FF00FF
    v = (v | (v >> 8)) & 0x0000FFFF0000FFFF
    v = (v | (v >> 16)) & 0x00000000FFFFFFFF
    return v


def encode_points(x, y, rect: Rect, level: int) -> np.ndarray:
    """Host Morton encode (geometry.py:105-135), used by validate() only."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = 1 << level
    tx = (x - rect.x_lo) / rect.width if rect.width > 0 else np.zeros_like(x)
    ty = (y - rect.y_lo) / rect.height if rect.height > 0 else np.zeros_like(y)
    cx = np.clip(np.floor(tx * n), 0, n - 1).astype(np.int64)
    cy = np.clip(np.floor(ty * n), 0, n - 1).astype(np.int64)
    return _spread(cx) | (_spread(cy) << 1)


def cell_bounds_arrays(levels, codes, mbr: Rect):
    """geometry.py:166-181."""
    levels = np.asarray(levels, dtype=np.int32)
    codes = np.asarray(codes, dtype=np.int64)
    cx, cy = _compact(codes), _compact(codes >> 1)
    return (
        mbr.x_lo + np.ldexp(cx.astype(np.float64), -levels) * mbr.width,
        mbr.y_lo + np.ldexp(cy.astype(np.float64), -levels) * mbr.height,
        mbr.x_lo + np.ldexp((cx + 1).astype(np.float64), -levels) * mbr.width,
        mbr.y_lo + np.ldexp((cy + 1).astype(np.float64), -levels) * mbr.height,
    )


@dataclass
class QuadIndex:
    """Immutable leaf grid sorted by Morton order key (quadindex.py:23-38)."""

    mbr: Rect
    th_quad: int
    l_max: int
    l_deep: int
    leaf_level: np.ndarray  # int32
    leaf_code: np.ndarray  # int64
    leaf_key: np.ndarray  # int64
    leaf_span: np.ndarray  # int64
    z_map: np.ndarray  # int32, 4**l_deep
    build_counts: np.ndarray  # int64
    n_build: int
    overfull_leaves: int

    @property
    def n_leaves(self) -> int:
        return len(self.leaf_level)

    def locate_codes(self, codes: np.ndarray) -> np.ndarray:
        return self.z_map[codes]

    def locate_points(self, x, y) -> np.ndarray:
        return self.z_map[encode_points(x, y, self.mbr, self.l_deep)]

    def validate(self, rng: np.random.Generator | None = None, probes: int = 10000) -> None:
        """Structural invariants (quadindex.py:51-76); AssertionError on violation."""
        spans = self.leaf_span
        n_codes = 4 ** self.l_deep
        assert int(spans.sum()) == n_codes, "leaf spans do not cover the code space"
        assert len(self.z_map) == n_codes
        starts = np.concatenate(([0], np.cumsum(spans)[:-1]))
        assert np.array_equal(starts, self.leaf_key), "leaf intervals overlap or leave gaps"
        below = self.leaf_level < self.l_max
        assert (self.build_counts[below] <= self.th_quad).all(), "leaf above l_max exceeds th_quad"
        if rng is None:
            rng = np.random.default_rng(0)
        px = rng.uniform(self.mbr.x_lo, self.mbr.x_hi, probes)
        py = rng.uniform(self.mbr.y_lo, self.mbr.y_hi, probes)
        ords = self.locate_points(px, py)
        x_lo, y_lo, x_hi, y_hi = cell_bounds_arrays(
            self.leaf_level[ords], self.leaf_code[ords], self.mbr)
        inside = (x_lo <= px) & (px <= x_hi) & (y_lo <= py) & (py <= y_hi)
        assert inside.all(), f"locate() disagrees with containment on {int((~inside).sum())} probes"


def should_rebuild(eval_counts, window: int = 3, factor: float = 1.5) -> bool:
    """quadindex.py:231-246 (the engine applies the same rule natively)."""
    counts = list(eval_counts)
    if window < 1:
        raise ValueError("window must be >= 1")
    if len(counts) < window + 1:
        return False
    last = counts[-1]
    trailing = counts[-window - 1: -1]
    return last > factor * (sum(trailing) / window)
