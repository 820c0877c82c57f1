"""Executed SASS instructions by opcode (and the source lines issuing a chosen
opcode set) from an `ncu --page source --csv --print-source=cuda,sass` dump."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
want = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else {"MUFU", "I2F", "F2I", "I2FP", "F2FP", "POPC", "FLO", "BREV"}
rows = list(csv.reader(open(path)))
ops = defaultdict(float)
by_line = defaultdict(float)
cur = None
src = {}
fname = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Function Name"):
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        src[cur] = r[1][:70]
        continue
    if r[0] == "" and len(r) > 7 and r[3]:
        txt = r[3].strip()
        if txt.startswith("@"):
            txt = txt.split(None, 1)[1] if " " in txt else txt
        op = txt.split()[0] if txt else "?"
        base = op.split(".")[0]
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        ops[base] += n
        if base in want and cur:
            by_line[cur] += n
tot = sum(ops.values())
print(f"total warp instructions {tot:.0f}")
for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:30]:
    print(f"  {k:10s} {v:10.0f}  {100 * v / tot:5.1f}%")
print("lines issuing", sorted(want))
for k, v in sorted(by_line.items(), key=lambda kv: -kv[1])[:25]:
    print(f"  {k[0]}:{k[1]:5d} {v:9.0f}  {src.get(k, '')}")
