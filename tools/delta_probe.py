"""Delta-tick timing probe (dev tool): update U objects then query."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
snap = synth.place(n, "uniform", seed=3)
qi, qx, qy = synth.queries(snap, n // 10, seed=3)
T = lambda a: torch.as_tensor(a, device="cuda")
dq = [T(qi), T(qx), T(qy)]
with Engine(EngineConfig(k=32, region=synth.REGION)) as eng:
    eng.load(snap.ids, snap.x, snap.y)
    out = eng.query_device(*dq)
    for frac in (0.0, 0.001, 0.01, 0.1, 0.3):
        for it in range(3):
            u = synth.updates(snap, frac, it, seed=3) if frac else (snap.ids[:0], snap.x[:0], snap.y[:0])
            du = [T(a) for a in u]
            torch.cuda.synchronize()
            t = time.perf_counter()
            if frac:
                eng.update(*du)
            out = eng.query_device(*dq, out=out)
            torch.cuda.synchronize()
            m = eng.last_metrics
        print(f"frac {frac}: wall {1e3*(time.perf_counter()-t):.2f} ms idxobj {m.t_index_objects_us} us")
