"""Aggregate an ncu 'cuda,sass' source page CSV per source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or not r[0].isdigit():
        continue
    d = dict(zip(hdr[:], r))
    try:
        inst = int(d["Instructions Executed"] or 0)
        samp = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    if inst or samp:
        out.append((samp, inst, cur_file, r[0], r[1][:70]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s} total inst {tot_i:.3e}")
for o in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*o[0]/tot_s:5.1f}% samp {100*o[1]/tot_i:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
