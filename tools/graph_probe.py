import sys, time, torch, numpy as np
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth
snap = synth.place(1_000_000, "uniform", seed=0)
qi, qx, qy = synth.queries(snap, 100_000, seed=1)
dev = torch.device("cuda:0")
T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
rng = np.random.default_rng(0)
with Engine(EngineConfig(k=32, region=synth.REGION)) as eng:
    eng.load(snap.ids, snap.x, snap.y)
    dq = [T(qi), T(qx), T(qy)]
    ups = []
    for b in range(4):
        sel = rng.choice(len(snap.ids), 100_000, replace=False)
        ups.append((T(snap.ids[sel]), T(snap.x[sel] + 1.0), T(snap.y[sel])))
    out = None
    for i in range(30):
        torch.cuda.synchronize(); t = time.perf_counter()
        eng.update(*ups[i % 4])
        out = eng.query_device(*dq, out=out)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        if i % 5 == 4: print(i, round(dt * 1e6), eng.graph_stats, eng.last_metrics.t_index_objects_us, (eng.last_metrics.t_first_iteration_us + eng.last_metrics.t_loop_us))
