"""ATOMIC scatter time vs where its scratch lands: a dummy cudaMalloc of
argv[1] MB is made before the library allocates its plan (one process per size)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth

cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
mb = float(sys.argv[1])
import paper_1404_1521_b200 as pg
rows, cols, N = 100_000, 64, 1_000_000
dist = os.environ.get("DIST", "zipf")
I, Y = synth.scatter_inputs(rows, cols, N, dist, "random", seed=42)
Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
W = torch.zeros(rows, cols, device="cuda")
fl = torch.empty(128 * 1024 * 1024, device="cuda")
torch.cuda.synchronize()
dummy = ctypes.c_void_p()
if mb > 0:
    ctypes.CDLL("libcudart.so").cudaMalloc(ctypes.byref(dummy), ctypes.c_size_t(int(mb * (1 << 20))))
pg.pg_scatter_add(W, Yd, Id, mode=1)   # the plan is allocated here
t = []
for _ in range(20):
    fl.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pg.pg_scatter_add_async(W, Yd, Id, mode=1)
    b.record()
    t.append((a, b))
torch.cuda.synchronize()
us = [a.elapsed_time(b) * 1e3 for a, b in t]
print(f"dummy {mb:6.2f} MB: {dist} atomic mean {statistics.mean(us):6.2f} us  median {statistics.median(us):6.2f}")
if os.environ.get("SHOW"):
    print("   per call:", " ".join(f"{x:.1f}" for x in us))
