"""Host-side value types of the drop-in boundary.

``Rect`` / ``Point`` keep the reference's semantics
(reference pkg/src/mknn/geometry.py:21-58): a closed axis-aligned rectangle,
finite coordinates, not inverted; ``width``/``height`` are evaluated as
``x_hi - x_lo`` in fp64 on the host and passed to the device unchanged so
Morton normalisation divides by bit-identical values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Point:
    x: float
    y: float


@dataclass(frozen=True)
class Rect:
    """Axis-aligned rectangle, closed on all edges (geometry.py:27-58)."""

    x_lo: float
    y_lo: float
    x_hi: float
    y_hi: float

    def __post_init__(self) -> None:
        vals = (self.x_lo, self.y_lo, self.x_hi, self.y_hi)
        if not all(math.isfinite(float(v)) for v in vals):
            raise ValueError("rect coordinates must be finite")
        if self.x_lo > self.x_hi or self.y_lo > self.y_hi:
            raise ValueError(f"inverted rect: {self}")

    @classmethod
    def square(cls, side: float, x_lo: float = 0.0, y_lo: float = 0.0) -> "Rect":
        return cls(x_lo, y_lo, x_lo + side, y_lo + side)

    @property
    def width(self) -> float:
        return self.x_hi - self.x_lo

    @property
    def height(self) -> float:
        return self.y_hi - self.y_lo

    def center(self) -> Point:
        return Point((self.x_lo + self.x_hi) / 2.0, (self.y_lo + self.y_hi) / 2.0)

    def contains(self, x: float, y: float) -> bool:
        return self.x_lo <= x <= self.x_hi and self.y_lo <= y <= self.y_hi
