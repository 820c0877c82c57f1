"""Per-CTA phase stamps of the cooperative radix sort (libpg_trace.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PG_LIB_VARIANT"] = "trace"
import numpy as np
import torch

import paper_1404_1521_b200 as pg
import synth

rows, cols, N = 100_000, 64, 1_000_000
I, Y = synth.scatter_inputs(rows, cols, N, sys.argv[1] if len(sys.argv) > 1 else "zipf", "random", seed=42)
Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
W = torch.zeros(rows, cols, device="cuda")
fl = torch.empty(128 * 1024 * 1024, device="cuda")
out = np.zeros((160, 16), dtype=np.uint64)
L = pg.lib()
for rep in range(3):
    fl.zero_()
    torch.cuda.synchronize()
    pg.pg_scatter_add(W, Yd, Id, mode=0)
    torch.cuda.synchronize()
L.pg_debug_sort_trace(out.ctypes.data_as(ctypes.c_void_p))
G = (N + 8191) // 8192
x = out[:G].astype(np.float64)
t0 = x[:, 0].min()
names = ["start", "p0.rank", "p0.cnt", "p0.bar1", "p0.bar2", "p0.scat", "p0.bar3", "p1.rank", "p1.cnt", "p1.bar1", "p1.bar2", "p1.scat"]
for k, nm in enumerate(names):
    col = (x[:, k] - t0) / 1e3
    print(f"{nm:8s} med {np.median(col):7.2f}  max {col.max():7.2f} us")
