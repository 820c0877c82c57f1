"""Executed SASS bytes per step.cu stage from an ncu source CSV (--print-source=cuda,sass)."""
import csv
import sys
from collections import defaultdict
sys.path.insert(0, __file__.rsplit('/', 1)[0])
path = sys.argv[1]
stages = [("gather_rows", 336, 380), ("agg_insert", 189, 224), ("agg_reset", 80, 96), ("fwd", 494, 522),
          ("sigma", 523, 593), ("bwd", 594, 623), ("record", 412, 466), ("aggregate", 226, 314),
          ("p1 other", 382, 628), ("dense", 1040, 1125), ("det_counts", 1408, 1444), ("p2prep", 1446, 1459),
          ("det_issue", 1461, 1499), ("det_merge", 1500, 1706), ("phase2", 1738, 1851), ("kernel", 2142, 2180)]
rows = list(csv.reader(open(path)))
hdr = None; cur = None; ln = None
addrs = defaultdict(set)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); continue
    if hdr is None:
        continue
    if r[0].isdigit():
        ln = int(r[0]); continue
    if r[0] == "" and r[2].startswith("0x"):
        try:
            ex = float(r[ie] or 0)
        except ValueError:
            ex = 0
        if ex <= 0:
            continue
        name = cur
        if cur == "step.cu":
            for nm, a, b in stages:
                if a <= ln <= b:
                    name = nm; break
        addrs[name].add(r[2])
tot = sum(len(v) for v in addrs.values()) * 16
print(f"executed code {tot / 1024:.1f} KB")
for k, v in sorted(addrs.items(), key=lambda kv: -len(kv[1])):
    print(f"  {k:28s} {len(v) * 16 / 1024:6.2f} KB")
