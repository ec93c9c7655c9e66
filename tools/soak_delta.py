"""Soak test (dev tool): many delta ticks (1 % and 10 % updates, incremental
and full re-index paths) against full-snapshot ticks of a second engine and
the brute-force certificate."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth
from paper_1412_6170_b200.verify import certify

n, nq, k, ticks = 1_000_000, 100_000, 32, int(sys.argv[1]) if len(sys.argv) > 1 else 60
snap = synth.place(n, "gaussian", seed=7, hotspots=8, sigma=900.0)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
bad = 0
with Engine(EngineConfig(k=k, region=synth.REGION)) as delta, \
        Engine(EngineConfig(k=k, region=synth.REGION)) as full:
    delta.load(snap.ids, snap.x, snap.y)
    for t in range(ticks):
        frac = 0.01 if t % 3 else 0.10
        ups = synth.updates(snap, frac, t, seed=7)
        synth.apply_updates(snap, *ups)
        delta.update(*ups)
        qi, qx, qy = synth.queries(snap, nq, seed=1000 + t)
        a = delta.query(qi, qx, qy)
        b = full.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        same = (np.array_equal(a.neighbour_ids, b.neighbour_ids)
                and a.distances.tobytes() == b.distances.tobytes()
                and delta.last_metrics.distance_evals == full.last_metrics.distance_evals
                and delta.last_metrics.rebuild_flag == full.last_metrics.rebuild_flag)
        if t % 10 == 9:
            d = [T(v) for v in (snap.ids, snap.x, snap.y, qi, qx, qy)]
            out = full.tick_device(*d)
            cert = certify(*d, k, out)
            same = same and all(v == 0 for v in cert.values())
        bad += not same
        if not same or t % 10 == 9:
            print(f"tick {t}: frac {frac} same {same} rebuild {delta.last_metrics.rebuild_flag}", flush=True)
print("soak bad ticks:", bad)
