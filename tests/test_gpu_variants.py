"""The measured alternatives behind the A/B switches compute
the same results as the default path: each runs in its own process (the
switches are read once per process) over the same ticks, and its digest of
rows, distances and metrics must equal the default's.  Among them is the
staged own-leaf pass (k_own1: cp.async.bulk leaf stages)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1412_6170_b200 import Engine, EngineConfig, synth
h = hashlib.sha256()
for k in (16, 32):
    snap = synth.place(200_000, "gaussian", seed=9, hotspots=6, sigma=600.0)
    x, y = snap.x.copy(), snap.y.copy()
    rng = np.random.default_rng(3)
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        out = None
        for t in range(4):
            if t:
                x = np.clip(x + rng.normal(0, 4.0, len(x)), 0, 22500)
                y = np.clip(y + rng.normal(0, 4.0, len(y)), 0, 22500)
            qi, qx, qy = synth.queries(synth.Snapshot(snap.ids, x, y), 20_000, seed=t)
            d = [torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")
                 for a in (snap.ids, x, y, qi, qx, qy)]
            out = eng.tick_device(*d, out=out)
            torch.cuda.synchronize()
            n = out["n_results"]
            for key in ("query_ids", "lengths", "offsets"):
                h.update(out[key].cpu().numpy().tobytes())
            h.update(out["neighbour_ids"][:n].cpu().numpy().tobytes())
            h.update(out["distances"][:n].cpu().numpy().tobytes())
            m = eng.last_metrics
            h.update(repr((m.distance_evals, m.pruned_leaves, m.active_left, m.active_right,
                           m.rebuild_flag)).encode())
print(h.hexdigest())
"""


def _digest(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


@pytest.fixture(scope="module")
def default_digest():
    return _digest({})


@pytest.mark.parametrize("switch", ["MKNN_OWN_STAGED=1", "MKNN_SEARCH_V0=1", "MKNN_GRAPH=0",
                                    "MKNN_BSORT=0", "MKNN_ONEPASS=0", "MKNN_BATCH=8"])
def test_variant_equals_default(switch, default_digest):
    name, value = switch.split("=")
    assert _digest({name: value}) == default_digest
