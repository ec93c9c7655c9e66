"""Host-side overhead of Engine.process_tick around the C call (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth

snap = synth.place(10_000_000, "gaussian", seed=3)
qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
k = 32
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
hs = [pin(a) for a in (snap.ids, snap.x, snap.y)]
hq = [pin(a) for a in (qi, qx, qy)]
nq = len(qi)
out = (torch.empty(nq, dtype=torch.int64).pin_memory().numpy(),
       torch.empty(nq, dtype=torch.int32).pin_memory().numpy(),
       torch.empty(nq * k, dtype=torch.int64).pin_memory().numpy(),
       torch.empty(nq * k, dtype=torch.float64).pin_memory().numpy(),
       np.empty(nq + 1, np.int64))
with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
    for it in range(6):
        t = time.perf_counter()
        res = eng.process_tick(*hs, *hq, out=out)
        w = (time.perf_counter() - t) * 1e6
        print(f"wall {w:.0f} us, engine total {eng.last_metrics.t_total_us} us, "
              f"host overhead {w - eng.last_metrics.t_total_us:.0f} us")

if len(sys.argv) > 1:
    import cProfile, pstats
    with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
        eng.process_tick(*hs, *hq, out=out)
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(5):
            eng.process_tick(*hs, *hq, out=out)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
