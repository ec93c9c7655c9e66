"""Aggregate an ncu 'cuda,sass' source CSV into named line ranges of mknn_search.cu.
usage: python tools/ncu_funcs.py x.csv"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
src = open("paper_1412_6170_b200/csrc/mknn_search.cu").read().split("\n")
# function starts: lines that open a definition at column 0 (device functions / kernels)
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"^(?:__device__|__global__|template|int |void |struct )", l)
    if m:
        name = re.search(r"(\w+)\s*\(", l) or re.search(r"struct (\w+)", l)
        if name:
            starts.append((i, name.group(1)))
def fn(line):
    best = "?"
    for s, n in starts:
        if s <= line: best = n
    return best
agg = {}
cur = hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].isdigit(): continue
    d = dict(zip(hdr, r))
    try:
        inst = int(d["Instructions Executed"] or 0); samp = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    key = fn(int(r[0])) if cur == "mknn_search.cu" else cur
    a = agg.setdefault(key, [0, 0]); a[0] += samp; a[1] += inst
ts = sum(a[0] for a in agg.values()) or 1; ti = sum(a[1] for a in agg.values()) or 1
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst ({i:.3e})  {k}")
