"""Executed-code footprint and no-instruction stalls by source region, from an
`ncu --page source --csv --print-source=cuda,sass` dump (instruction-cache study)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
gran = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rows = list(csv.reader(open(path)))
cur = None; fname = None; hdr = None
static = defaultdict(int); execd = defaultdict(int); noinst = defaultdict(float); samp = defaultdict(float)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        d = dict(zip(hdr, r))
        k = (cur[0], cur[1] // gran * gran)
        try:
            noinst[k] += float(d.get("stall_no_inst") or 0)
            samp[k] += float(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            pass
        continue
    if r[0] == "" and len(r) > 7 and r[3] and cur:
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        k = (cur[0], cur[1] // gran * gran)
        static[k] += 1
        if n > 0:
            execd[k] += 1
te = sum(execd.values()); ts = sum(samp.values()); tn = sum(noinst.values())
print(f"executed code {te * 16 / 1024:.1f} KB of {sum(static.values()) * 16 / 1024:.1f} KB; "
      f"samples {ts:.0f}, no_inst {tn:.0f} ({100 * tn / max(ts, 1):.1f}%)")
for k in sorted(static):
    if execd[k] > 20 or noinst[k] > 5:
        print(f"  {k[0]:>28s}:{k[1]:5d}  exec {execd[k] * 16 / 1024:5.1f} KB  samples {samp[k]:5.0f}  no_inst {noinst[k]:4.0f}")
