"""Per-CTA phase stamps of the ATOMIC scatter kernel sc_atomic_hot (libpg_trace.so)."""
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
for dist in (sys.argv[1:] or ["zipf", "uniform"]):
    I, Y = synth.scatter_inputs(rows, cols, N, dist, "random", seed=42)
    Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
    W = torch.zeros(rows, cols, device="cuda")
    fl = torch.empty(128 * 1024 * 1024, device="cuda")
    out = np.zeros((160, 16), dtype=np.uint64)
    L = pg.lib()
    for rep in range(3):
        fl.zero_()
        torch.cuda.synchronize()
        pg.pg_scatter_add(W, Yd, Id, mode=1)
        torch.cuda.synchronize()
    L.pg_debug_sort_trace(out.ctypes.data_as(ctypes.c_void_p))
    x = out[:148].astype(np.float64)
    t0 = x[:, 0].min()
    names = ["start", "validated", "hotset", "bar.wait", "stream.end", "sync", "tierA.flush", "bar2", "end", "Wprefetch", "hashinit", "samplehash", "candsorted", "cand.own", "cand.sync"]
    print(dist)
    for k, nm in enumerate(names):
        col = np.where(x[:, k] > 0, (x[:, k] - t0) / 1e3, np.nan)
        if np.isnan(col).all():
            continue
        print(f"  {nm:11s} med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
    last = out[:148, 15].astype(np.uint64)
    if last.any():   # slot 15: the last warp to finish the candidate extraction (warp << 56 | time)
        wl = (last >> np.uint64(56)).astype(int)
        tl = (last & np.uint64((1 << 56) - 1)).astype(np.float64)
        print("  last warp at the candidate barrier: warp ids", np.bincount(wl, minlength=32).nonzero()[0].tolist(),
              f"med {np.median((tl - t0) / 1e3):.2f} us")
