"""Where does the e2e tick time go? (dev tool)"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth
from paper_1412_6170_b200 import _native as N

snap = synth.place(10_000_000, "gaussian", seed=3)
qi, qx, qy = synth.queries(snap, 1_000_000, seed=3)
k = 32
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
h = [pin(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
d = [t.cuda() for t in h]
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    for a, b in zip(d, h):
        a.copy_(b, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D 264 MB pinned: {(time.perf_counter()-t)/3*1e3:.2f} ms")
out_d = torch.empty(1_000_000 * k * 2, dtype=torch.float64, device="cuda")
out_h = torch.empty(1_000_000 * k * 2, dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    out_h.copy_(out_d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H 512 MB pinned: {(time.perf_counter()-t)/3*1e3:.2f} ms")
hn = [a.numpy() for a in h]
outs = (torch.empty(1_000_000, dtype=torch.int64).pin_memory().numpy(),
        torch.empty(1_000_000, dtype=torch.int32).pin_memory().numpy(),
        torch.empty(1_000_000 * k, dtype=torch.int64).pin_memory().numpy(),
        torch.empty(1_000_000 * k, dtype=torch.float64).pin_memory().numpy())
import ctypes
lib = N.lib()
with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
    for it in range(4):
        t = time.perf_counter()
        res = eng.process_tick(*hn, out=outs)
        t1 = time.perf_counter()
        m = eng.last_metrics
        print(f"process_tick pinned: {1e3*(t1-t):.2f} ms (engine total {m.t_total_us} us, "
              f"idx {m.t_index_objects_us}, search {(m.t_first_iteration_us + m.t_loop_us)})")
    t = time.perf_counter()
    o = eng.tick_device(*d)
    torch.cuda.synchronize()
    print(f"tick_device: {1e3*(time.perf_counter()-t):.2f} ms")
