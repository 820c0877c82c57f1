"""Per-function / per-line stall breakdown from an ncu source CSV (cuda,sass view)."""
import csv
import sys
from collections import defaultdict

path, srcfile = sys.argv[1], sys.argv[2]
fns = sys.argv[3:]
rows = list(csv.reader(open(path)))
hdr = None; cur = None
agg = defaultdict(lambda: defaultdict(float)); txt = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (cur, int(r[0])); txt[key] = r[1][:70]
    for i, hn in enumerate(hdr):
        if i >= len(r):
            break
        if hn.startswith("stall_") or hn in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[key][hn] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
src = open(srcfile).read().split('\n')
base = srcfile.split('/')[-1]


def rng(name):
    for i, l in enumerate(src):
        if name in l:
            j = i
            while j < len(src) and not src[j].startswith('}'):
                j += 1
            return i + 1, j + 1
    return None


for fn in fns:
    ab = rng(fn)
    if not ab:
        continue
    a, b = ab
    items = [(k, v) for k, v in agg.items() if k[0] == base and a <= k[1] <= b]
    s = sum(v["Warp Stall Sampling (All Samples)"] for k, v in items)
    ins = sum(v["Instructions Executed"] for k, v in items)
    print(f"== {fn} lines {a}-{b}: stall {100 * s / tot:.1f}%  inst {ins / 148:.0f}/SM")
    for k, v in sorted(items, key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:8]:
        st = sorted([(x, n) for n, x in v.items() if n.startswith('stall_') and 'Not Issued' not in n], reverse=True)[:3]
        print(f"   {k[1]:4d} {100 * v['Warp Stall Sampling (All Samples)'] / tot:5.1f}% inst/SM {v['Instructions Executed'] / 148:7.0f}  "
              f"{txt[k]}  | " + ", ".join(f"{n[6:]}:{x:.0f}" for x, n in st))
