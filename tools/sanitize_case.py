"""Small ticks for compute-sanitizer (dev tool): full, delta, sliced-host, k>32."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, Rect, synth

rng = np.random.default_rng(1)
snap = synth.place(20_000, "gaussian", seed=2, hotspots=3)
qi, qx, qy = synth.queries(snap, 3_000, seed=2)
for k in (8, 32, 100):
    with Engine(EngineConfig(k=k, region=synth.REGION)) as e:
        r = e.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
        e.load(snap.ids, snap.x, snap.y)
        for t in range(3):
            e.update(*synth.updates(snap, 0.1, t, seed=3))
            r = e.query(qi, qx, qy)
        print("k", k, "ok", r.neighbour_ids[:3])
big = synth.place(100_000, "uniform", seed=5)
bq = synth.queries(big, 70_000, seed=5)
with Engine(EngineConfig(k=16, region=synth.REGION)) as e:
    r = e.process_tick(big.ids, big.x, big.y, *bq)
    print("sliced ok", r.lengths[:3])
