"""Stall samples and executed SASS bytes per step.cu function (ranges from the current
source) from an ncu source CSV (ncu -i rep --page source --csv --print-source=cuda,sass)."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
src = open(sys.argv[2] if len(sys.argv) > 2 else "paper_1404_1521_b200/csrc/step.cu").read().split("\n")
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))
# inside phase1_fast, split by stage comments
for i, l in enumerate(src, 1):
    for key, nm in (("// ---- forward partials", "p1.forward"), ("// ---- sigma stage", "p1.sigma"),
                    ("// ---- backward:", "p1.backward"), ("auto write_record", "p1.record")):
        if key in l:
            starts.append((i, nm))
starts.sort()


def fn_of(ln):
    name = "?"
    for s, nm in starts:
        if s <= ln:
            name = nm
        else:
            break
    return name


rows = list(csv.reader(open(path)))
hdr = None
cur = None
ln = None
agg = defaultdict(lambda: defaultdict(float))
code = defaultdict(set)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        ln = int(r[0])
        name = fn_of(ln) if cur == "step.cu" else cur
        for i, hn in enumerate(hdr):
            if i >= len(r):
                break
            if (hn.startswith("stall_") and "Not Issued" not in hn) or hn in ("Warp Stall Sampling (All Samples)",):
                try:
                    agg[name][hn] += float(r[i] or 0)
                except ValueError:
                    pass
        continue
    if r[0] == "" and len(r) > 2 and r[2].startswith("0x"):
        try:
            if float(r[ie] or 0) > 0:
                code[fn_of(ln) if cur == "step.cu" else cur].add(r[2])
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
print(f"| region | warp samples | executed SASS | top stall reasons |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"]):
    s = v["Warp Stall Sampling (All Samples)"]
    if s < 0.01 * tot:
        continue
    st = sorted([(x, n) for n, x in v.items() if n.startswith("stall_")], reverse=True)[:3]
    print(f"| {k} | {100 * s / tot:.1f} % | {len(code[k]) * 16 / 1024:.1f} KB | " +
          ", ".join(f"{n[6:]} {100 * x / s:.0f} %" for x, n in st) + " |")
print(f"\nexecuted SASS total: {sum(len(v) for v in code.values()) * 16 / 1024:.1f} KB")
