"""Small ticks for compute-sanitizer (dev tool): full, delta, sliced-host, k>32 (32-bit and 64-bit merge keys)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, Rect, synth

rng = np.random.default_rng(1)
snap = synth.place(20_000, "gaussian", seed=2, hotspots=3)
qi, qx, qy = synth.queries(snap, 3_000, seed=2)
for k in (8, 32, 100, 300):
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
# steady-state device ticks: one-pass partition, bucket sort, graph replay
import torch
d = [torch.as_tensor(np.ascontiguousarray(a), device="cuda:0") for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
with Engine(EngineConfig(k=32, region=synth.REGION)) as e:
    out = None
    for t in range(5):
        out = e.tick_device(*d, out=out)
    torch.cuda.synchronize()
    print("device ticks ok", e.graph_stats)
# 1M objects: balanced partition buckets -> bucket-local sort (two-pass on the
# rebuild tick, one-pass after), graph replay; a delta tick sequence
mid = synth.place(1_000_000, "uniform", seed=7)
mq = synth.queries(mid, 100_000, seed=7)
dm = [torch.as_tensor(np.ascontiguousarray(a), device="cuda:0") for a in (mid.ids, mid.x, mid.y, *mq)]
with Engine(EngineConfig(k=32, region=synth.REGION)) as e:
    out = None
    for t in range(4):
        out = e.tick_device(*dm, out=out)
    torch.cuda.synchronize()
    e.load(mid.ids, mid.x, mid.y)
    for t in range(3):
        e.update(*synth.updates(mid, 0.1, t, seed=4))
        r = e.query(*mq)
    print("1M ticks ok", e.graph_stats, r.lengths[:3])
