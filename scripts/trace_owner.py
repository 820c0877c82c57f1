"""Per-CTA phase stamps of the DET owner-bucket scatter kernel (libpg_trace.so)."""
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
noflush = "--noflush" in sys.argv
for dist in ([a for a in sys.argv[1:] if not a.startswith("--")] or ["zipf", "uniform"]):
    I, Y = synth.scatter_inputs(rows, cols, N, dist, "random", seed=42)
    Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
    W = torch.zeros(rows, cols, device="cuda")
    fl = torch.empty(128 * 1024 * 1024, device="cuda")
    out = np.zeros((160, 16), dtype=np.uint64)
    L = pg.lib()
    for rep in range(3):
        if not noflush:
            fl.zero_()
        torch.cuda.synchronize()
        pg.pg_scatter_add(W, Yd, Id, mode=0)
        torch.cuda.synchronize()
    L.pg_debug_owner_trace(out.ctypes.data_as(ctypes.c_void_p))
    x = out[:148].astype(np.float64)
    t0 = x[:, 0].min()
    names = ["start", "A.hotset", "A.arrive", "H.sorted", "A.wait", "B.arrive", "C.start", "C.sorted", "C.end", "D.end", "A.loaded", "A.sampled", "B.Hload", "B.count", "A.tagged", "A.passed"]
    print(dist, "(no flush)" if noflush else "(L2 flushed)")
    for k, nm in enumerate(names):
        col = np.where(x[:, k] > 0, (x[:, k] - t0) / 1e3, np.nan)
        if np.isnan(col).all():
            continue
        print(f"  {nm:9s} med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
