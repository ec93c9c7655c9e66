"""Summarise one ncu --set full capture for profiles/.
usage: python tools/ncu_summary.py rep.ncu-rep [algorithmic_bytes_per_launch] > profiles/<name>.txt"""
import csv, io, subprocess, sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}
for vals in rows[2:]:
    d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    print(f"== {d.get('Kernel Name', '?')[:100]}")
    for k in KEYS[1:]:
        if k in d:
            print(f"  {k:60s} {d[k]} {u[k]}")
    rd = num(d.get("dram__bytes_read.sum", "")) or 0
    wr = num(d.get("dram__bytes_write.sum", "")) or 0
    tr = (rd * SCALE.get(u.get("dram__bytes_read.sum"), 1) + wr * SCALE.get(u.get("dram__bytes_write.sum"), 1))
    t = num(d.get("gpu__time_duration.sum", "")) * SCALE.get(u.get("gpu__time_duration.sum"), 1)
    print(f"  traffic (dram read+write) bytes/launch                       {tr:.4g}")
    if alg:
        print(f"  algorithmic bytes/launch                                     {alg:.4g} "
              f"(achieved {alg / t / 1e9:.1f} GB/s over the ncu duration)")
    st = {h[len('smsp__pcsamp_warps_issue_stalled_'):]: num(v) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(v for v in st.values() if v) or 1
    print("  warp-stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                                              sorted(st.items(), key=lambda kv: -(kv[1] or 0))[:8] if v))
