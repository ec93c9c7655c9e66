"""DESIGN.md §5 results rows from bench lines (gpurun_out/matrix/<wl>.json or
profiles/r2_bench_<wl>.json).  usage: python tools/results_table.py [dir] [prefix]"""
import json, os, sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/matrix"
pre = sys.argv[2] if len(sys.argv) > 2 else ""
ROUND1 = {"cfg2": "146.8M (0.681 ms)", "cfg3": "312.4M (3.201 ms)", "cfg3u": "326.8M",
          "cfg4": "345.4M (29.0 ms)", "k1": "572.5M", "k8": "441.5M", "k32": "311.4M",
          "k128": "54.7M (18.3 ms)"}
NAME = {"cfg2": "cfg2: uniform 1M, 100K q, k=32, 10% updates/tick (delta)",
        "cfg3": "**cfg3: Gaussian/16 10M, 1M q, k=32 (headline; default `python bench.py`)**",
        "cfg3u": "cfg3 variant: uniform 10M, 1M q, k=32",
        "cfg4": "cfg4: uniform 100M, 10M q, k=16, 10% updates/tick (1 GPU)",
        "k1": "cfg5: Gaussian/16 10M, 1M q, k=1", "k8": "cfg5: k=8", "k32": "cfg5: k=32",
        "k128": "cfg5: k=128"}
for wl in ("cfg2", "cfg3", "cfg3u", "cfg4", "k1", "k8", "k32", "k128"):
    p = os.path.join(d, f"{pre}{wl}.json")
    if not os.path.exists(p):
        continue
    b = json.load(open(p))
    ph = b["tick_phases_us"]
    ms = b["ms_per_step"]
    tick = f"{ms:.3f} ms" if ms < 10 else f"{ms:.2f} ms"
    q = f"{b['value'] / 1e6:.1f}M"
    if wl == "cfg3":
        q, tick = f"**{q}**", f"**{tick}**"
    e2e = f"{b['e2e']['value'] / 1e6:.1f}M"
    print(f"| {NAME[wl]} | {q} | {tick} | {b['roofline']['frac']:.3f} | "
          f"{b['roofline']['tick_frac']:.3f} | {ph['index_objects']} / {ph['index_queries']} / "
          f"{ph['search']} / {ph['emit']} | {'**' + e2e + '**' if wl == 'cfg3' else e2e} | {ROUND1[wl]} |")
