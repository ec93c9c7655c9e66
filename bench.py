#!/usr/bin/env python
"""Benchmark of the per-tick repeated k-NN join (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload cfg3|cfg3u|cfg2|cfg2s|cfg4|cfg4s|k1|k8|k32|k128]

A step is one tick -> every query's k nearest (id, distance) lists, CSR in
issuer order.  Snapshot workloads (cfg3, cfg3u, k*, cfg2s, cfg4s) hand the
engine the full position snapshot every tick; delta workloads (cfg2, cfg4:
BASELINE.json's "10% position updates per tick") hand it the tick's U
position updates over the device-resident snapshot (carry-forward semantics
of datasets.py:136-148).
Default workload (the metric is quoted "at 10M objects"): BASELINE.json
configs[2], Gaussian-clustered n=10M (16 hotspots, sigma 500), 1M queries,
k=32; synthetic data from the reference generator's placement draws
(paper_1412_6170_b200/synth.py).

* value: queries/s of the whole job with inputs resident in HBM
  (Engine.tick_device, or Engine.update + Engine.query_device for delta
  workloads), timed with CUDA events per step on the launching stream, L2
  flushed between steps outside the timed events, max over ranks.
* e2e: the same metric through the reference-facing API (Engine.process_tick
  -> C-ABI mknn_tick, or Engine.update + Engine.query) with pinned HOST
  buffers: the H2D of the snapshot or updates and the queries and the D2H of
  the result CSR are inside every timed step.
* roofline: the dominant kernel (k_search); algorithmic bytes per launch =
  24*T + 24*Q + 16*Q*k (T = records the reference's distance tasks stream,
  counted on device in one extra untimed instrumented step), divided by the
  kernel's CUDA-event time (engine metrics t_first_iteration_us + t_loop_us:
  the one search kernel's time, split by its batches' own-leaf warp time).
* cpu_baseline: the C port of the reference engine (oracle/, OpenMP, all host
  threads) on a steady-state tick (index reused) with a bounded query sample,
  scaled to one tick.
* --impl reference: the same port, every step a full steady-state tick with
  all queries, plus the threads=1 port figure and the unmodified Python
  reference (mknn.Engine from baseline/_ref) on bounded samples.
* --gpus N>1 (torchrun): strong scaling by default (the workload's query
  batch split over the ranks, BASELINE configs[3]); --scaling weak gives
  every rank the full batch.  The snapshot (or the tick's updates) arrive as
  1/N slices per rank and are all-gathered over NCCL every step
  (sharded.py); the replicated re-index and the query phase are reported
  separately.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-NN queries/sec per tick at 10M objects, 1/2/4/8 B200; % of HBM roofline"
UNIT = "queries/s"

WORKLOADS = {
    "cfg3": dict(desc="Gaussian-clustered 10M objects (16 hotspots, sigma 500), 1M queries, k=32",
                 dist="gaussian", n=10_000_000, nq=1_000_000, k=32, seed=3, baseline_idx=2),
    "cfg3u": dict(desc="uniform 10M objects, 1M queries, k=32", dist="uniform", n=10_000_000,
                  nq=1_000_000, k=32, seed=3, baseline_idx=2),
    "cfg2": dict(desc="uniform 1M objects, 100K queries, k=32, 10% position updates per tick",
                 dist="uniform", n=1_000_000, nq=100_000, k=32, seed=0, baseline_idx=1,
                 updates=0.10),
    "cfg2s": dict(desc="uniform 1M objects, 100K queries, k=32, full snapshot per tick",
                  dist="uniform", n=1_000_000, nq=100_000, k=32, seed=0, baseline_idx=1),
    "cfg4": dict(desc="uniform 100M objects, 10M queries, k=16, 10% position updates per tick",
                 dist="uniform", n=100_000_000, nq=10_000_000, k=16, seed=4, baseline_idx=3,
                 updates=0.10),
    "cfg4s": dict(desc="uniform 100M objects, 10M queries, k=16, full snapshot per tick",
                  dist="uniform", n=100_000_000, nq=10_000_000, k=16, seed=4, baseline_idx=3),
}
for _k in (1, 8, 32, 128):
    WORKLOADS[f"k{_k}"] = dict(desc=f"Gaussian-clustered 10M objects, 1M queries, k={_k}",
                               dist="gaussian", n=10_000_000, nq=1_000_000, k=_k, seed=3,
                               baseline_idx=4)


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~2 ms on a
    background thread during the timed region (the timed region is only tens
    of ms, shorter than nvidia-smi's sampling period)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = None

    def _run(self, h, pynvml):
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis else self.gpu
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, args=(h, pynvml), daemon=True)
            self._t.start()
        except Exception:
            self._stop = None
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted(nm for nm, bit in self.REASONS.items()
                         if any(rs & bit for _, rs in self.samples))
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def cpu_port_tick_seconds(snap, qi, qx, qy, k, region, th, sample_q, index=None):
    """The C port of the reference engine (oracle/, test infrastructure used
    here only as the reported CPU baseline), as a steady-state tick: the
    index built on an earlier tick is reused (engine.py:615-619), so a step
    is index_objects + index_queries + the distance phases + emission.  The
    query part runs on ``sample_q`` queries and is scaled to the tick.
    Returns (seconds per tick, seconds of the object re-index, seconds of the
    sampled tick, threads)."""
    from oracle import oracle as orc

    own = index is None
    if own:
        index = orc.build_index(snap.x, snap.y, region, th, 10)
    try:
        t = time.perf_counter()
        orc.engine_tick(snap.ids, snap.x, snap.y, qi[:0], qx[:0], qy[:0], k, region, th,
                        index=index)
        t_index = time.perf_counter() - t
        if sample_q >= len(qi):
            t = time.perf_counter()
            orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, k, region, th, index=index)
            t_sample = time.perf_counter() - t
            return t_sample, t_index, t_sample, orc.num_threads()
        t = time.perf_counter()
        orc.engine_tick(snap.ids, snap.x, snap.y, qi[:sample_q], qx[:sample_q], qy[:sample_q], k,
                        region, th, index=index)
        t_sample = time.perf_counter() - t
    finally:
        if own:
            orc.free_index(index)
    per_q = max(t_sample - t_index, 0.0) / max(sample_q, 1)
    return t_index + per_q * len(qi), t_index, t_sample, orc.num_threads()


def python_reference_tick_seconds(snap, qi, qx, qy, k, region, sample_q, threads):
    """The reference package itself (mknn.Engine from baseline/_ref, the
    unmodified pure-Python/numpy engine, engine.py:557-701) on a steady-state
    tick: a first tick builds the index, a 0-query tick times the per-tick
    object re-index, a ``sample_q``-query tick the per-query part, scaled to
    the full query count.  None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mknn")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from mknn import Engine as RefEngine, EngineConfig as RefConfig, Rect as RefRect

    r = RefRect(region.x_lo, region.y_lo, region.x_hi, region.y_hi)
    s = slice(0, sample_q)
    with RefEngine(RefConfig(k=k, region=r, threads=threads)) as eng:
        eng.process_tick(snap.ids, snap.x, snap.y, qi[:0], qx[:0], qy[:0])  # builds the index
        t = time.perf_counter()
        eng.process_tick(snap.ids, snap.x, snap.y, qi[:0], qx[:0], qy[:0])
        t0 = time.perf_counter() - t
        t = time.perf_counter()
        eng.process_tick(snap.ids, snap.x, snap.y, qi[s], qx[s], qy[s])
        t1 = time.perf_counter() - t
        assert eng.last_metrics.rebuild_flag == 0
    per_q = max(t1 - t0, 0.0) / max(min(sample_q, len(qi)), 1)
    return dict(value=len(qi) / (t0 + per_q * len(qi)), unit=UNIT, cores=threads,
                kind="reference",
                sample=f"mknn.Engine (baseline/_ref) threads={threads}: steady-state tick over "
                       f"{len(snap.ids)} objects with 0 queries ({t0:.2f} s) and {sample_q} "
                       f"queries ({t1:.2f} s), scaled to {len(qi)} queries")


def make_inputs(wl, world=1, rank=0, strong=True):
    """The workload's snapshot and this rank's queries: strong scaling
    splits the workload's query batch over the ranks, weak scaling gives
    every rank a batch of that size."""
    from paper_1412_6170_b200 import synth

    snap = synth.place(wl["n"], wl["dist"], seed=wl["seed"])
    nq_total = min(wl["nq"] * (1 if strong else world), wl["n"])
    qi, qx, qy = synth.queries(snap, nq_total, seed=wl["seed"])
    if world > 1:
        from paper_1412_6170_b200.sharded import shard_queries

        sel = shard_queries(qi, world, rank)
        qi, qx, qy = qi[sel], qx[sel], qy[sel]
    return snap, qi, qx, qy


def config_of(wl, nq_total, world, scaling, th, delta, U):
    """The ``config`` object of both arms' JSON lines (same keys)."""
    return {
        "workload": wl["desc"], "baseline_config": wl["baseline_idx"], "n_objects": wl["n"],
        "n_queries": int(nq_total), "k": wl["k"], "th_quad": th, "l_max": 10,
        "parallelism": (f"query shards x{world} ({scaling} scaling), replicated index, NCCL "
                        f"all-gather of {'update' if delta else 'snapshot'} slices")
        if world > 1 else "single GPU",
        "l2": "flushed between steps (256 MB write outside the timed events); "
              "inputs 264 MB > 126 MB L2",
        "updates_per_tick": int(U) if delta else None,
    }


def run_reference(args, wl):
    """--impl reference: the reference's CPU algorithm -- the C port of its
    engine (oracle/, OpenMP over all host threads) -- on the same workload:
    every step is a full steady-state tick (all queries; the index built on
    the first tick is reused, engine.py:615-619).  Rank 0 only.  The line
    also carries the threads=1 port figure and the unmodified Python
    reference (baseline/_ref) timed on bounded samples."""
    from oracle import oracle as orc
    from paper_1412_6170_b200 import synth
    from paper_1412_6170_b200.engine import resolve_th_quad

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    snap, qi, qx, qy = make_inputs(wl)
    th = resolve_th_quad("auto", wl["k"])
    # every host thread (torchrun sets OMP_NUM_THREADS=1 per process; rank 0
    # alone runs this arm, so it may use the whole host)
    orc.set_num_threads(os.cpu_count() or 1)
    index = orc.build_index(snap.x, snap.y, synth.REGION, th, 10)  # the first tick's rebuild
    for _ in range(args.warmup):  # warm-up: the re-index and a small query batch
        cpu_port_tick_seconds(snap, qi, qx, qy, wl["k"], synth.REGION, th, 1000, index=index)
    secs = []
    for _ in range(args.steps):
        t = time.perf_counter()
        orc.engine_tick(snap.ids, snap.x, snap.y, qi, qx, qy, wl["k"], synth.REGION, th,
                        index=index)
        secs.append(time.perf_counter() - t)
    threads = orc.num_threads()
    ms = 1e3 * statistics.mean(secs)
    value = len(qi) / (ms / 1e3)
    extra = {}
    if not args.no_cpu_extras:
        orc.set_num_threads(1)
        s1, _, _, _ = cpu_port_tick_seconds(snap, qi, qx, qy, wl["k"], synth.REGION, th,
                                            min(len(qi), 20_000), index=index)
        orc.set_num_threads(threads)
        extra["port_threads_1"] = {"value": len(qi) / s1, "unit": UNIT, "cores": 1, "kind": "port",
                                   "sample": "steady-state tick, 20000 queries scaled"}
        for nt in (os.cpu_count() or 1, 1):
            r = python_reference_tick_seconds(snap, qi, qx, qy, wl["k"], synth.REGION,
                                              2_000 if nt == 1 else 10_000, nt)
            if r is not None:
                extra[f"python_reference_threads_{nt}"] = r
    orc.free_index(index)
    delta = bool(wl.get("updates"))
    U = int(round(wl["n"] * wl["updates"])) if delta else wl["n"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling_of(args), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(wl, len(qi), args.gpus, scaling_of(args), th, delta, U),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"every step a full steady-state tick: {wl['n']} objects "
                                   f"re-indexed, all {len(qi)} queries (oracle/mknn_oracle.c, "
                                   f"OpenMP over {threads} threads; index built once, as on the "
                                   f"reference's non-rebuild ticks)",
                         **({"extra": extra} if extra else {})},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def scaling_of(args) -> str:
    return "weak" if args.scaling == "weak" else "strong"


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-sample", type=int, default=250_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-extras", action="store_true",
                    help="--impl reference: skip the threads=1 and Python-reference figures")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = the workload's queries split over the ranks "
                         "(BASELINE configs[3]), weak = that many queries per rank")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    from paper_1412_6170_b200 import Engine, EngineConfig, synth
    from paper_1412_6170_b200 import _native
    from paper_1412_6170_b200.engine import resolve_th_quad

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MKNN_BENCH_BACKEND=gloo: every rank on cuda:0 with gloo collectives (a
    # functional check of the N > 1 path on a one-GPU box; never a bench value)
    backend = os.environ.get("MKNN_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    k = wl["k"]
    th = resolve_th_quad("auto", k)

    strong = args.scaling == "strong"
    snap, qi, qx, qy = make_inputs(wl, world, rank, strong)
    nq = len(qi)
    nq_job = torch.tensor([nq], dtype=torch.int64, device=dev)
    lo, hi = (0, wl["n"])
    if world > 1:
        from paper_1412_6170_b200.sharded import ShardedEngine, shard_bounds

        lo, hi = shard_bounds(wl["n"], world, rank)
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    d_qi, d_qx, d_qy = T(qi), T(qx), T(qy)
    cfg = EngineConfig(k=k, region=synth.REGION, device=local)
    stream = torch.cuda.current_stream(dev)
    delta = bool(wl.get("updates"))
    if world > 1:
        eng = ShardedEngine(cfg, local)
        engine = eng.engine
    else:
        engine = Engine(cfg)
        engine.set_stream(stream)
    if delta:
        # tick = the tick's U position updates (datasets.py:136-148 carry-forward
        # over the device-resident snapshot) + the query batch; a few distinct
        # update batches are cycled (the last update per id wins)
        n_batches = 4
        batches = [synth.updates(snap, wl["updates"], t, seed=wl["seed"]) for t in range(n_batches)]
        U = len(batches[0][0])
        ulo, uhi = shard_bounds(U, world, rank) if world > 1 else (0, U)
        d_up = [(T(b[0][ulo:uhi]), T(b[1][ulo:uhi]), T(b[2][ulo:uhi])) for b in batches]
        if world > 1:
            eng.load_slices(T(snap.ids[lo:hi]), T(snap.x[lo:hi]), T(snap.y[lo:hi]), n_total=wl["n"])
            step = lambda out, i: eng.update_tick_device(*d_up[i % n_batches], d_qi, d_qx, d_qy,  # noqa: E731
                                                         out=out, n_total=U)
        else:
            engine.load(snap.ids, snap.x, snap.y)

            def step(out, i):
                engine.update(*d_up[i % n_batches])
                return engine.query_device(d_qi, d_qx, d_qy, out=out)
    else:
        U = wl["n"]
        d_ids, d_x, d_y = T(snap.ids[lo:hi]), T(snap.x[lo:hi]), T(snap.y[lo:hi])
        if world > 1:
            step = lambda out, i: eng.tick_device(d_ids, d_x, d_y, d_qi, d_qx, d_qy, out=out,  # noqa: E731
                                                  n_total=wl["n"])
        else:
            step = lambda out, i: engine.tick_device(d_ids, d_x, d_y, d_qi, d_qx, d_qy, out=out)  # noqa: E731
    out = engine.alloc_device_out(nq, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    for i in range(args.warmup):
        step(out, i)
    torch.cuda.synchronize(dev)

    # one extra untimed, instrumented step: T for the roofline
    engine.instrument = True
    step(out, 0)
    T_records = engine.last_streamed_records
    engine.instrument = False
    step(out, 1)
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    search_us, tick_metrics = [], []
    launches0 = _native.lib().mknn_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the timed events
            ev[i][0].record(stream)
            step(out, i)
            ev[i][1].record(stream)
            m = engine.last_metrics
            search_us.append(m.t_first_iteration_us + m.t_loop_us)
            tick_metrics.append(m)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    launches = _native.lib().mknn_kernel_launches() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.all_reduce(nq_job)
    ms_per_step = float(t_local.item()) / args.steps
    nq_total = int(nq_job.item())
    value = nq_total / (ms_per_step / 1e3)
    # the replicated part (update ingest, re-index) against the
    # query phase (index_queries + search + emission), max over ranks
    ph = torch.tensor([statistics.mean(m.t_build_us + m.t_index_objects_us for m in tick_metrics),
                       statistics.mean(m.t_index_queries_us + m.t_first_iteration_us
                                       + m.t_loop_us + m.t_emit_us
                                       for m in tick_metrics)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    replicated_us, query_phase_us = (float(v) for v in ph.tolist())

    # ---- e2e through the reference-facing API with pinned host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        h_q = [pin(qi), pin(qx), pin(qy)]
        h_out = (torch.empty(nq, dtype=torch.int64).pin_memory().numpy(),
                 torch.empty(nq, dtype=torch.int32).pin_memory().numpy(),
                 torch.empty(nq * k, dtype=torch.int64).pin_memory().numpy(),
                 torch.empty(nq * k, dtype=torch.float64).pin_memory().numpy(),
                 np.empty(nq + 1, dtype=np.int64))
        if delta:
            h_up = [[pin(a[ulo:uhi]) for a in b] for b in batches]
            if world == 1:
                def e2e_step(i):
                    engine.update(*h_up[i % n_batches])
                    return engine.query(*h_q, out=h_out)
            else:
                e2e_step = lambda i: eng.update_tick(*h_up[i % n_batches], *h_q, n_total=U)  # noqa: E731
            h2d = 24 * (uhi - ulo) + 24 * nq
        else:
            h_snap = [pin(snap.ids[lo:hi]), pin(snap.x[lo:hi]), pin(snap.y[lo:hi])]
            if world == 1:
                e2e_step = lambda i: engine.process_tick(*h_snap, *h_q, out=h_out)  # noqa: E731
            else:
                e2e_step = lambda i: eng.process_tick(*h_snap, *h_q, n_total=wl["n"])  # noqa: E731
            h2d = 24 * (hi - lo) + 24 * nq
        e2e_step(0)  # warm the host path
        if world > 1:
            dist.barrier()
        secs, nres = [], 0
        for i in range(args.e2e_steps):
            t = time.perf_counter()
            res = e2e_step(i)
            secs.append(time.perf_counter() - t)
            nres = len(res.neighbour_ids)
        t_e2e = torch.tensor([statistics.mean(secs)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e = {"value": nq_total / float(t_e2e.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(12 * nq + 16 * nres)}

    # ---- roofline of the dominant kernel (k_search) -----------------------
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not peak:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    t_search_s = statistics.mean(search_us) / 1e6
    search_bytes = 24 * T_records + 24 * nq + 16 * nq * k
    achieved = search_bytes / t_search_s / 1e9
    # ncu --set full capture of the same kernel on the same workload (per launch)
    prof = (load_json(os.path.join(ROOT, "profiles", "search_kernel_traffic.json")) or {})
    prof = prof.get(args.workload, {}) if isinstance(prof, dict) else {}
    traffic = prof.get("traffic_bytes_per_launch")
    tick_bytes = 24 * U + 64 * wl["n"] + 48 * nq + 24 * T_records + 16 * nq * k
    m0 = tick_metrics[-1]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling_of(args), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(wl, nq_total, world, scaling_of(args), th, delta, U),
        "timed": ("Engine.update (U device-resident update records) + Engine.query_device per "
                  "step: update apply, rebuild decision, index_objects, index_queries, search, "
                  "emission to device CSR" if delta else
                  "Engine.tick_device per step: rebuild decision, index_objects, "
                  "index_queries, search, emission to device CSR"),
        "phases_max_over_ranks_us": {"replicated_reindex": replicated_us,
                                     "query_phase": query_phase_us,
                                     "queries_per_rank": nq},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": {
            "bound": "hbm", "kernel": "k_search", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_src,
            "bytes_per_launch": int(search_bytes),
            "bytes_formula": "24*T + 24*Q + 16*Q*k, T = streamed records counted on device",
            "T": int(T_records), "t_launch_us": t_search_s * 1e6,
            "tick_B_alg": int(tick_bytes),
            "tick_frac": tick_bytes / (ms_per_step / 1e3) / 1e9 / peak,
            # SURVEY §8(d) floor: T := n (every object streamed once)
            "tick_B_min": int(tick_bytes - 24 * T_records + 24 * wl["n"]),
            # secondary figures of the same kernel from its ncu capture
            "fp64_pipe_pct": prof.get("fp64_pipe_pct") if traffic else None,
            "issue_active_pct": prof.get("issue_active_pct") if traffic else None,
        },
        "clocks": clk.summary(),
        "tick_phases_us": {"build": m0.t_build_us, "index_objects": m0.t_index_objects_us,
                           "index_queries": m0.t_index_queries_us,
                           "search": m0.t_first_iteration_us + m0.t_loop_us,
                           "search_first_iteration": m0.t_first_iteration_us,
                           "emit": m0.t_emit_us},
        "tick_metrics": {"distance_evals": m0.distance_evals, "pruned_leaves": m0.pruned_leaves,
                         "iterations_left": m0.iterations_left,
                         "iterations_right": m0.iterations_right},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s, t_index, t_sample, threads = cpu_port_tick_seconds(
            snap, qi, qx, qy, k, synth.REGION, th, min(args.cpu_sample, nq))
        line["cpu_baseline"] = {
            "value": nq / s, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"C port of the reference engine (oracle/mknn_oracle.c), steady-state tick "
                      f"(index reused): re-index of {wl['n']} objects ({t_index:.2f} s) + "
                      f"{min(args.cpu_sample, nq)} of {nq} queries ({t_sample - t_index:.2f} s), "
                      f"scaled to {nq} queries"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
    else:
        engine.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
