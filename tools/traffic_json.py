"""Per-workload DRAM traffic of the dominant search kernel, from the ncu
summaries in profiles/ (tools/gpu_prof_r2.sh -> r2_search_ncu_<workload>.txt),
into profiles/search_kernel_traffic.json, which bench.py reads for
roofline.traffic.  usage: python tools/traffic_json.py [round-tag]"""
import json, os, re, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
out = {}
for wl in ("cfg2", "cfg3", "cfg3u", "cfg4", "k1", "k8", "k32", "k128"):
    src = os.path.join(ROOT, "profiles", f"{tag}_search_ncu_{wl}.txt")
    if wl == "k32" and not os.path.exists(src):  # k32 is the cfg3 workload
        src = os.path.join(ROOT, "profiles", f"{tag}_search_ncu_cfg3.txt")
    if not os.path.exists(src):
        continue
    txt = open(src).read()
    kern = re.search(r"^== (.*)$", txt, re.M).group(1).strip()
    def metric(name):
        m = re.search(rf"^\s+{re.escape(name)}\s+([0-9.,]+(?:e[+-]?[0-9]+)?)", txt, re.M)
        return float(m.group(1).replace(",", "")) if m else None
    out[wl] = {
        "kernel": kern,
        "traffic_bytes_per_launch": metric("traffic (dram read+write) bytes/launch"),
        "duration": " ".join(re.search(r"gpu__time_duration.sum\s+(\S+ \S+)", txt).group(1).split()),
        "fp64_pipe_pct": metric("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "source": f"profiles/{os.path.basename(src)}: ncu --set full --clock-control none, "
                  f"python bench.py --workload {wl} --steps 1 --warmup 3 (dram__bytes_read.sum + "
                  "dram__bytes_write.sum of one k_search launch)",
    }
json.dump(out, open(os.path.join(ROOT, "profiles", "search_kernel_traffic.json"), "w"), indent=1)
print(json.dumps({k: v["traffic_bytes_per_launch"] for k, v in out.items()}))
