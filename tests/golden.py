"""Loader for the fixtures written by tests/golden/make_golden.py (which runs
the real reference package).  Used by the CPU oracle tests and the GPU parity
tests alike; nothing here reads /root/reference at run time."""

from __future__ import annotations

import glob
import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from paper_1412_6170_b200.geometry import Rect

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def result_digest(res) -> str:
    return digest(np.asarray(res.query_ids, np.int64), np.asarray(res.lengths, np.int32),
                  np.asarray(res.neighbour_ids, np.int64), np.asarray(res.distances, np.float64))


@dataclass
class Tick:
    ids: np.ndarray
    x: np.ndarray
    y: np.ndarray
    qi: np.ndarray
    qx: np.ndarray
    qy: np.ndarray
    meta: dict
    arrays: dict

    def has(self, key):
        return key in self.arrays

    def __getitem__(self, key):
        return self.arrays[key]


@dataclass
class Case:
    name: str
    meta: dict
    ticks: list

    @property
    def region(self) -> Rect:
        return Rect(*self.meta["region"])

    @property
    def k(self) -> int:
        return int(self.meta["k"])

    @property
    def th_quad(self):
        return self.meta["th_quad"]

    @property
    def l_max(self) -> int:
        return int(self.meta["l_max"])


def load_case(path) -> Case:
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    ticks = []
    for t in range(meta["n_ticks"]):
        pre = f"t{t}_"
        arrays = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        ticks.append(Tick(arrays["ids"], arrays["x"], arrays["y"], arrays["qi"], arrays["qx"],
                          arrays["qy"], meta["ticks"][t], arrays))
    return Case(meta["name"], meta, ticks)


def case_paths():
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("cfg1"))


def case_names():
    return [os.path.basename(p)[:-4] for p in case_paths()]


def load(name) -> Case:
    return load_case(os.path.join(GOLDEN, name + ".npz"))


def load_cfg1():
    z = np.load(os.path.join(GOLDEN, "cfg1_uniform_100k.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return meta, {k: z[k] for k in z.files if k != "meta"}


def load_geometry():
    with open(os.path.join(GOLDEN, "geometry.json")) as f:
        return json.load(f)


def th_of(case: Case) -> int:
    th = case.th_quad
    if th == "auto":
        k = case.k
        return 192 if k < 32 else (12 * k if k <= 128 else 2048)
    return int(th)
