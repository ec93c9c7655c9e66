"""Time Engine.update on device tensors (dev tool): 100M snapshot, 10M updates."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
snap = synth.place(n, "uniform", seed=4)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
ups = [[T(a) for a in synth.updates(snap, 0.1, t, seed=4)] for t in range(3)]
with Engine(EngineConfig(k=16, region=synth.REGION)) as e:
    e.load(snap.ids, snap.x, snap.y)
    for it in range(6):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        a.record()
        e.update(*ups[it % 3])
        b.record()
        torch.cuda.synchronize()
        print(f"update: wall {(time.perf_counter() - t) * 1e3:.2f} ms, device {a.elapsed_time(b):.2f} ms")
