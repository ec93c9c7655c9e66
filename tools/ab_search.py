"""A/B of the search kernels on one workload (dev tool): prints search time
and a digest of the device results.  MKNN_SEARCH_V0=1 selects the round-1
kernel.  usage: python tools/ab_search.py dist n nq k [iters]"""
import hashlib, os, sys
import torch
sys.path.insert(0, ".")
from paper_1412_6170_b200 import Engine, EngineConfig, synth

dist, n, nq, k = sys.argv[1], int(float(sys.argv[2])), int(float(sys.argv[3])), int(sys.argv[4])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 5
snap = synth.place(n, dist, seed=3)
qi, qx, qy = synth.queries(snap, nq, seed=3)
dev = torch.device("cuda:0")
d = [torch.as_tensor(a, device=dev) for a in (snap.ids, snap.x, snap.y, qi, qx, qy)]
ts, ti = [], []
with Engine(EngineConfig(k=k, region=synth.REGION)) as eng:
    out = None
    for it in range(iters):
        out = eng.tick_device(*d, out=out)
        torch.cuda.synchronize()
        ts.append((eng.last_metrics.t_first_iteration_us + eng.last_metrics.t_loop_us))
        ti.append(eng.last_metrics.t_index_objects_us)
    m = eng.last_metrics
    h = hashlib.sha256()
    for key in ("query_ids", "lengths", "offsets", "neighbour_ids", "distances"):
        h.update(out[key].cpu().numpy().tobytes())
tag = "v0" if os.environ.get("MKNN_SEARCH_V0") == "1" else "v1"
tag += os.environ.get("AB_TAG", "")
print(f"{tag} {dist} n={n} nq={nq} k={k}: search us {sorted(ts)[len(ts)//2]} idx_obj us {sorted(ti)[len(ti)//2]} (all {ts}) "
      f"evals {m.distance_evals} prunes {m.pruned_leaves} digest {h.hexdigest()[:16]}", flush=True)
