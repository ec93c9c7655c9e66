"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv log.
usage: python tools/launch_summary.py launches.csv [n_ticks]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
ticks = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[h]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[h + 1:]:
    if len(r) <= vi: continue
    n = r[ki].split("(")[0].replace("mknn::<unnamed>::", "")
    agg[n][0] += 1; agg[n][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
tot = sum(a[1] for a in agg.values())
print(f"{'us/tick':>10} {'share':>6} {'launches':>8}  kernel")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / ticks:10.1f} {100 * t / tot:5.1f}% {c / ticks:8.1f}  {n[:90]}")
