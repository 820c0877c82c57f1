"""A few scatter-add calls (for ncu): python scripts/prof_scatter.py det|atomic zipf|uniform [calls]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1404_1521_b200 as pg
import synth

mode = {"det": 0, "atomic": 1}[sys.argv[1] if len(sys.argv) > 1 else "det"]
dist = sys.argv[2] if len(sys.argv) > 2 else "zipf"
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
I, Y = synth.scatter_inputs(100_000, 64, 1_000_000, dist, "random", seed=42)
Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
W = torch.zeros(100_000, 64, device="cuda")
for _ in range(calls):
    pg.pg_scatter_add(W, Yd, Id, mode=mode)
torch.cuda.synchronize()
print("ok")
