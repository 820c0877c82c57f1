"""Per-CTA phase timestamps of the fused step (PG_OPT_TRACE, libpg_trace.so), averaged over steps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PG_LIB_VARIANT"] = "trace"   # instrumented build: python -m paper_1404_1521_b200.build --trace
import numpy as np
import torch

import paper_1404_1521_b200 as pg
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--split", action="store_true")
ap.add_argument("--atomic", action="store_true")
ap.add_argument("--flush", action="store_true")
ap.add_argument("--busy", action="store_true", help="keep the GPU busy between steps (no host sync)")
ap.add_argument("--large", action="store_true", help="V 1M, d 128, n 5, h 128 (tiled path)")
a = ap.parse_args()
V, d, n, h = (1_000_000, 128, 5, 128) if a.large else (100_000, 64, 5, 32)
m = pg.PolyglotModel(V, d, n, h, fused=not a.split, scatter=1 if a.atomic else 0)
P = min(148, a.batch)
tr = torch.zeros(a.steps, 160 * 64, dtype=torch.int64, device="cuda")
bs = [synth.batch(V, n, a.batch, seed=1, step=t) for t in range(a.steps)]
di = [torch.from_numpy(i).cuda() for i, _ in bs]
dc = [torch.from_numpy(c).cuda() for _, c in bs]
fl = torch.empty(128 * 1024 * 1024, device="cuda")
for t in range(a.steps):
    pg.pg_set_option(m.handle, 5, tr[t].data_ptr())
    if a.flush:
        fl.zero_()
    m.train_step(di[t], dc[t], 0.1, loss_out=None)
    if not a.busy:
        torch.cuda.synchronize()
torch.cuda.synchronize()
names = ["start", "gathered", "fwd", "sigma", "bwd", "agg", "p1end", "barrier", "p2head", "dense", "", "end",
         "", "", "agg.ins", "agg.scan", "agg.place", "agg.acc", "agg.csr", "idx",
         "m.esrc", "m.trip2", "m.hash", "m.scan", "m.trip3", "g.rows", "w1", "s.loaded", "s.shfl", "p2.dense_ld", "p2.counts"]
X = tr.view(a.steps, 160, 64).cpu().numpy()[2:, :P].astype(np.float64)
rel = []
mhz = []
for x in X:
    t0 = x[:, 0].min()
    y = x[:, :31].copy()
    y[:, 12:14] = 0
    rel.append(np.where(y > 0, y - t0, np.nan))
    mhz.append(np.median((x[:, 13] - x[:, 12]) / (x[:, 11] - x[:, 0]) * 1e3))
A = np.stack(rel)
print(f"B={a.batch} split={a.split} flush={a.flush} busy={a.busy} SM clock in kernel ~{np.median(mhz):.0f} MHz "
      f"(us from earliest CTA start; median / max over CTAs)")
order = [0, 19, 25, 26, 1, 2, 27, 28, 3, 4, 14, 15, 16, 18, 17, 5, 6, 7, 29, 30, 8, 9, 20, 21, 22, 23, 24, 11]
for k in order:
    nm = names[k]
    col = A[:, :, k]
    if np.isnan(col).all():
        continue
    print(f"  {nm:9s} med {np.nanmedian(col) / 1e3:7.2f}  max {np.nanmean(np.nanmax(col, axis=1)) / 1e3:7.2f}")
G = {39: "g.start", 40: "g.stage0", 42: "g.stage1", 44: "g.stage2", 46: "g.comp", 47: "g.red", 48: "g.end"}
XG = tr.view(a.steps, 160, 64).cpu().numpy()[2:, :P].astype(np.float64)
for k, nm in G.items():
    col = XG[:, :, k]
    t0 = XG[:, :, 0].min(axis=1, keepdims=True)
    v = np.where(col > 0, col - t0, np.nan)
    if np.isnan(v).all():
        continue
    print(f"  {nm:9s} med {np.nanmedian(v) / 1e3:7.2f}  max {np.nanmean(np.nanmax(v, axis=1)) / 1e3:7.2f}")

# slowest CTAs (last step): end time, owner entry count M, per-stage deltas
x = X[-1]
t0 = x[:, 0].min()
ends = (x[:, 11] - t0) / 1e3
slow = np.argsort(-ends)[:6]
print("slowest CTAs (last step): cta end_us M | trip2 hash scan trip3 sums (us)")
for b in slow:
    st = [(x[b, k2] - x[b, k1]) / 1e3 for k1, k2 in ((20, 21), (21, 22), (22, 23), (23, 24), (24, 11))]
    print(f"  {b:4d} {ends[b]:6.2f} {int(x[b, 31]):4d} | " + " ".join(f"{v:5.2f}" for v in st))
    if x[b, 43] > 0:   # sorted fallback stamps: keys built, sorted, segments, windows done
        print("       fallback: start->keys {:5.2f} sort {:5.2f} segs {:5.2f} windows {:5.2f} | after {:5.2f}".format(
            (x[b, 40] - x[b, 29]) / 1e3, (x[b, 41] - x[b, 40]) / 1e3, (x[b, 42] - x[b, 41]) / 1e3,
            (x[b, 43] - x[b, 42]) / 1e3, (x[b, 11] - x[b, 43]) / 1e3))
        print("       first window: stage {:5.2f} sums {:5.2f}".format((x[b, 44] - x[b, 42]) / 1e3, (x[b, 45] - x[b, 44]) / 1e3))
        print("       window ends (us after segs):", " ".join("{:5.2f}".format((x[b, k] - x[b, 42]) / 1e3) for k in range(46, 50) if x[b, k] > 0))
        print("       per window staged / summed (us after segs):", " ".join("{:5.2f}".format((x[b, k] - x[b, 42]) / 1e3) for k in range(50, 58) if x[b, k] > 0))
med = np.median(X[-1][:, 31])
print(f"median M {med:.0f}, max M {X[-1][:, 31].max():.0f}")

if a.large:   # tiled path, second chunk (slots 32 + k)
    for k, nm in ((33, "c2.xt"), (34, "c2.fwd"), (35, "c2.sigma"), (59, "c2.G"), (36, "c2.dW1"), (37, "c2.agg")):
        col = A2 = (X[:, :, k] - X[:, :, 0].min(axis=1, keepdims=True)) / 1e3
        print(f"  {nm:9s} med {np.nanmedian(col):7.2f}  max {np.nanmean(np.nanmax(col, axis=1)):7.2f}")
