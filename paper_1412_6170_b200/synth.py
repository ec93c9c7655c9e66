"""Synthetic tick inputs for benches and tests (harness, not the hot path).

Placement restates the reference generator's draw order exactly so that
inputs are bit-identical on the same numpy (PCG64, NEP 19):
``WorkloadGenerator._place`` (reference pkg/src/mknn/workload.py:186-209):

* uniform:  x = rng.uniform(x_lo, x_hi, n); y = rng.uniform(y_lo, y_hi, n)
* gaussian: hotspot centres cx, cy ~ uniform(hotspots) each, object i joins
  hotspot i % hotspots, offsets ~ normal(0, sigma) for x then y, clipped.

Queries follow SURVEY.md §8(d): issuers are
``default_rng(seed + 1).choice(n, Q, replace=False)`` and each query sits at
its issuer's position.

The per-tick update stream (cfg 2/4: a 10 % sample of objects moves) is a
harness construct the reference does not ship; its movement here is a
bounded uniform step reflected into the region (our own, documented in
DESIGN.md), since only the update *rate* matters for the measurement.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Rect

REGION = Rect.square(22500.0)  # workload.py:37 default region


@dataclass
class Snapshot:
    ids: np.ndarray
    x: np.ndarray
    y: np.ndarray


def place(n: int, distribution: str = "uniform", seed: int = 0, hotspots: int = 16,
          sigma: float = 500.0, region: Rect = REGION) -> Snapshot:
    rng = np.random.default_rng(seed)
    ids = np.arange(n, dtype=np.int64)
    r = region
    if distribution == "uniform":
        x = rng.uniform(r.x_lo, r.x_hi, n)
        y = rng.uniform(r.y_lo, r.y_hi, n)
    elif distribution == "gaussian":
        cx = rng.uniform(r.x_lo, r.x_hi, hotspots)
        cy = rng.uniform(r.y_lo, r.y_hi, hotspots)
        which = ids % hotspots
        x = cx[which] + rng.normal(0.0, sigma, n)
        y = cy[which] + rng.normal(0.0, sigma, n)
        x = np.clip(x, r.x_lo, r.x_hi)
        y = np.clip(y, r.y_lo, r.y_hi)
    else:
        raise ValueError(f"unknown distribution {distribution!r}")
    return Snapshot(ids, x, y)


def queries(snap: Snapshot, nq: int, seed: int = 0):
    """(q_issuer, qx, qy): nq distinct issuers at their own positions."""
    n = len(snap.ids)
    nq = min(nq, n)
    sel = np.random.default_rng(seed + 1).choice(n, nq, replace=False)
    return snap.ids[sel].copy(), snap.x[sel].copy(), snap.y[sel].copy()


def updates(snap: Snapshot, frac: float, tick: int, seed: int = 0, max_speed: float = 200.0,
            region: Rect = REGION):
    """A seeded ``frac`` sample of objects with new positions (one tick of
    movement).  Returns (ids, x, y) of the updated objects."""
    n = len(snap.ids)
    u = int(round(n * frac))
    rng = np.random.default_rng([seed, 7919, tick])
    sel = rng.choice(n, u, replace=False)
    step = rng.uniform(-max_speed, max_speed, (2, u)) * np.sqrt(0.5)
    nx = _reflect(snap.x[sel] + step[0], region.x_lo, region.x_hi)
    ny = _reflect(snap.y[sel] + step[1], region.y_lo, region.y_hi)
    return snap.ids[sel].copy(), nx, ny


def apply_updates(snap: Snapshot, uid, ux, uy) -> None:
    """Carry-forward semantics (reference datasets.py:136-148) for ids that
    equal their array position (ids = arange(n))."""
    snap.x[uid] = ux
    snap.y[uid] = uy


def _reflect(v, lo, hi):
    v = np.where(v < lo, 2 * lo - v, v)
    v = np.where(v > hi, 2 * hi - v, v)
    return np.clip(v, lo, hi)
