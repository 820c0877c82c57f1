"""Run a few Polyglot SGD steps (for ncu / nsight launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1404_1521_b200 as pg
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--split", action="store_true")
ap.add_argument("--atomic", action="store_true")
ap.add_argument("--scatter-bench", action="store_true")
ap.add_argument("--large", action="store_true", help="V 1M, d 128, n 5, h 128 (tiled path)")
a = ap.parse_args()
V, d, n, h = (1_000_000, 128, 5, 128) if a.large else (100_000, 64, 5, 32)
if a.scatter_bench:
    I, Y = synth.scatter_inputs(V, d, 1_000_000, "zipf", "random")
    W = torch.zeros(V, d, device="cuda")
    Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
    for _ in range(a.steps):
        pg.pg_scatter_add(W, Yd, Id, mode=1 if a.atomic else 0)
    torch.cuda.synchronize()
    sys.exit(0)
m = pg.PolyglotModel(V, d, n, h, seed=42, fused=not a.split, scatter=1 if a.atomic else 0)
bs = [synth.batch(V, n, a.batch, seed=1, step=t) for t in range(a.steps)]
di = [torch.from_numpy(i).cuda() for i, _ in bs]
dc = [torch.from_numpy(c).cuda() for _, c in bs]
for t in range(a.steps):
    m.train_step(di[t], dc[t], 0.1, loss_out=None)
torch.cuda.synchronize()
m.sync()
print("ok")
