"""Quick device timing of one workload (dev tool; bench.py is the contract)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth

dist = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10_000_000
nq = int(float(sys.argv[3])) if len(sys.argv) > 3 else 1_000_000
k = int(sys.argv[4]) if len(sys.argv) > 4 else 32
t0 = time.time()
snap = synth.place(n, dist, seed=3)
qi, qx, qy = synth.queries(snap, nq, seed=3)
print(f"gen {time.time()-t0:.1f}s", flush=True)
dev = torch.device("cuda:0")
T = lambda a: torch.as_tensor(a, device=dev)
d = [T(a) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
    out = None
    for it in range(int(__import__("os").environ.get("QT_ITERS", "6"))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = eng.tick_device(*d, out=out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        m = eng.last_metrics
        print(f"it {it}: wall {dt*1e3:.2f} ms build {m.t_build_us} idxobj {m.t_index_objects_us} "
              f"idxq {m.t_index_queries_us} search {(m.t_first_iteration_us + m.t_loop_us)} emit {m.t_emit_us} us; "
              f"evals/q {m.distance_evals/nq:.1f} prunes/q {m.pruned_leaves/nq:.1f} "
              f"iters {m.iterations_left}/{m.iterations_right} rebuild {m.rebuild_flag}", flush=True)
    ix = eng.index
    print("l_deep", ix.l_deep, "leaves", ix.n_leaves, "overfull", ix.overfull_leaves)
    t = time.perf_counter()
    res = eng.process_tick(snap.ids, snap.x, snap.y, qi, qx, qy)
    print(f"host-path tick (pageable) {1e3*(time.perf_counter()-t):.1f} ms")
