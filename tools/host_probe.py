"""Host-side cost of a device tick (dev tool): wall time of tick_device,
of the C call alone, of _finish, against the device phases."""
import sys, time, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth, _native as N
from paper_1412_6170_b200 import engine as E

n, nq, k = int(float(sys.argv[1])), int(float(sys.argv[2])), int(sys.argv[3])
snap = synth.place(n, "gaussian", seed=3)
qi, qx, qy = synth.queries(snap, nq, seed=3)
dev = torch.device("cuda:0")
d = [torch.as_tensor(a, device=dev) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
orig_finish = Engine._finish
acc = {"finish": []}
def timed_finish(self, m):
    t = time.perf_counter(); r = orig_finish(self, m); acc["finish"].append(time.perf_counter() - t); return r
Engine._finish = timed_finish
with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
    out = None
    for i in range(25):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); e0.record()
        out = eng.tick_device(*d, out=out)
        e1.record(); wall = time.perf_counter() - t
        torch.cuda.synchronize()
        m = eng.last_metrics
        if i >= 20:
            ph = m.t_build_us + m.t_index_objects_us + m.t_index_queries_us + (m.t_first_iteration_us + m.t_loop_us) + m.t_emit_us
            print(f"wall {wall*1e6:.0f} us, events {e0.elapsed_time(e1)*1e3:.0f} us, phases {ph} us, "
                  f"C total {m.t_total_us} us, _finish {acc['finish'][-1]*1e6:.0f} us, graph {eng.graph_stats}")
