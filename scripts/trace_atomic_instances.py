"""ATOMIC scatter stage stamps for several instances of libpg_trace.so in one
process (each with its own scratch allocation): where does the Zipf time of a
slow instance go?  python scripts/trace_atomic_instances.py N"""
import ctypes
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth

here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1404_1521_b200")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
libs = []
for k in range(N):
    path = f"/tmp/libpg_trace_{k}.so"
    shutil.copy(os.path.join(here, "libpg_trace.so"), path)
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    L.pg_scatter_add_async.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, ctypes.c_int64, ctypes.c_int, P, P]
    L.pg_debug_sort_trace.argtypes = [P]
    libs.append(L)
rows, cols, n = 100_000, 64, 1_000_000
I, Y = synth.scatter_inputs(rows, cols, n, "zipf", "random", seed=42)
Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
W = torch.zeros(rows, cols, device="cuda")
fl = torch.empty(128 * 1024 * 1024, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
names = ["start", "validated", "hotset", "bar.wait", "stream.end", "sync", "tierA.flush", "bar2", "end"]
for k, L in enumerate(libs):
    acc = []
    for rep in range(6):
        fl.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.pg_scatter_add_async(W.data_ptr(), rows, cols, Yd.data_ptr(), Id.data_ptr(), n, 1, s, None)
        b.record()
        torch.cuda.synchronize()
        out = np.zeros((160, 16), dtype=np.uint64)
        L.pg_debug_sort_trace(out.ctypes.data_as(ctypes.c_void_p))
        x = out[:148, :9].astype(np.float64)
        x = (x - x[:, 0].min()) / 1e3
        if rep >= 2:
            acc.append((a.elapsed_time(b) * 1e3, np.median(x, axis=0), x.max(axis=0)))
    ev = np.mean([t for t, _, _ in acc])
    med = np.mean([m for _, m, _ in acc], axis=0)
    mx = np.mean([m for _, _, m in acc], axis=0)
    print(f"instance {k}: event {ev:6.1f} us | " + " ".join(f"{nm} {med[i]:5.1f}/{mx[i]:5.1f}" for i, nm in enumerate(names)))
