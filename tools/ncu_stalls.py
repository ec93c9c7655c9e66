"""Per-source-line stall breakdown from an ncu 'cuda,sass' source CSV.
usage: python tools/ncu_stalls.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        tot = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    if not tot:
        continue
    key = (cur, r[0], r[1][:60])
    st = {h[6:]: int(d[h] or 0) for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
    a = agg.setdefault(key, [0, {}])
    a[0] += tot
    for kk, v in st.items():
        a[1][kk] = a[1].get(kk, 0) + v
T = sum(v[0] for v in agg.values())
for key, (tot, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100*tot/T:5.1f}%  {key[0]}:{key[1]:<5} {key[2]:<60} " +
          " ".join(f"{k}={100*v/tot:.0f}%" for k, v in top if v))
