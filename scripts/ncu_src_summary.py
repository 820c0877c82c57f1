"""Summarise an `ncu --page source --csv --print-source=cuda,sass` dump by CUDA source line."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
cur_file = None
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[:2], r[:2]))
    try:
        samples = float(r[4] or 0)
        inst = float(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    agg[key][0] += samples
    agg[key][1] += inst
    agg[key][2] = r[1][:90]
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:4d}  stall {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_i:5.1f}%  {v[2]}")
