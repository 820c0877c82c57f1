"""Stall samples per step.cu stage (line ranges) from an ncu source CSV (--print-source=cuda,sass)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
stages = [("gather_rows", 336, 380), ("agg_insert", 189, 224), ("agg_reset", 80, 96), ("fwd", 494, 522),
          ("sigma", 523, 593), ("bwd", 594, 623), ("record", 412, 466), ("aggregate", 226, 314),
          ("p1 other", 382, 628), ("dense", 1040, 1125), ("det_counts", 1408, 1444), ("p2prep", 1446, 1459),
          ("det_issue", 1461, 1499), ("det_merge", 1500, 1706), ("phase2", 1738, 1851), ("kernel", 2142, 2180)]
rows = list(csv.reader(open(path)))
hdr = None
cur = None
agg = defaultdict(lambda: defaultdict(float))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    ln = int(r[0])
    name = cur
    if cur == "step.cu":
        for nm, a, b in stages:
            if a <= ln <= b:
                name = nm
                break
    for i, hn in enumerate(hdr):
        if i >= len(r):
            break
        if (hn.startswith("stall_") and "Not Issued" not in hn) or hn in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[name][hn] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
print(f"total samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"]):
    s = v["Warp Stall Sampling (All Samples)"]
    if s < 0.005 * tot:
        continue
    st = sorted([(x, n) for n, x in v.items() if n.startswith("stall_")], reverse=True)[:5]
    print(f"{k:14s} {100 * s / tot:5.1f}%  inst/SM {v['Instructions Executed'] / 148:8.0f}  " +
          ", ".join(f"{n[6:]}:{100 * x / s:.0f}%" for x, n in st))
