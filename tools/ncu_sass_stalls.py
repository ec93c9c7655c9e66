"""Top SASS instructions by long-scoreboard stall and the load feeding them.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_sass_stalls.py x.csv [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        recs.append((r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix["stall_long_sb"]] or 0),
                     int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0)))
    except ValueError:
        pass
tot = sum(x[3] for x in recs) or 1
lsb = sum(x[2] for x in recs) or 1
print(f"samples {tot}, long_sb {lsb} ({100*lsb/tot:.1f}%)")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
pos = {x[0]: i for i, x in enumerate(recs)}
for a, src, l, s, e in sorted(recs, key=lambda x: -x[2])[:n]:
    i = pos[a]
    # nearest preceding global/local loads
    loads = [recs[j][1] for j in range(max(0, i - 40), i) if recs[j][1].split()[0].lstrip("@!P0123456789 ").startswith(("LDG", "LD.", "LDL", "LD "))]
    print(f"{100*l/lsb:5.1f}% lsb  {src[:60]:60s}  <- {loads[-2:] if loads else ''}")
