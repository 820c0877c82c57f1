"""Same-process A/B of scatter-add variants: python scripts/ab_scatter.py MODE LIB [LIB ...]
(LIB = 'main' for paper_1404_1521_b200/libpg.so, or a path from scripts/ab_variant.py).
Every round runs each library once, in a rotating order, on the same buffers,
L2 flushed before each call; prints the mean and median event time per library.

CAVEAT: each library instance allocates its own scratch, and the ATOMIC Zipf
time depends on where that lands (76-88 us by placement), so
the list position biases the comparison; compare one library per process at
controlled placements instead (scripts/place_scan.py, PG_LIB_PATH)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth

mode = {"det": 0, "atomic": 1}[sys.argv[1]]
names = sys.argv[2:]
here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1404_1521_b200")
libs = []
for nm in names:
    L = ctypes.CDLL(os.path.join(here, "libpg.so") if nm == "main" else nm)
    P = ctypes.c_void_p
    L.pg_scatter_add_async.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, ctypes.c_int64, ctypes.c_int, P, P]
    L.pg_scatter_add_async.restype = ctypes.c_int
    libs.append(L)
rows, cols, N = 100_000, 64, 1_000_000
rounds = int(os.environ.get("ROUNDS", "30"))
flush = torch.empty(128 * 1024 * 1024, device="cuda")
for dist in ("zipf", "uniform"):
    I, Y = synth.scatter_inputs(rows, cols, N, dist, "random", seed=42)
    U = int(np.unique(I).size)
    alg = N * (4 * cols + 4) + 2 * U * 4 * cols
    Id, Yd = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
    W = torch.zeros(rows, cols, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    call = lambda L: L.pg_scatter_add_async(W.data_ptr(), rows, cols, Yd.data_ptr(), Id.data_ptr(), N, mode, s, None)
    for L in libs:
        assert call(L) == 0
    ev = {k: [] for k in range(len(libs))}
    block = int(os.environ.get("BLOCK", "1"))   # consecutive calls of one library per round
    for r in range(rounds):
        for j in range(len(libs)):
            k = (j + r) % len(libs)
            for _ in range(block):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                call(libs[k])
                b.record()
                ev[k].append((a, b))
    torch.cuda.synchronize()
    for k, nm in enumerate(names):
        t = [a.elapsed_time(b) * 1e3 for a, b in ev[k]]
        m = statistics.mean(t)
        print(f"{dist:8s} {os.path.basename(nm):22s} mean {m:7.2f} us  median {statistics.median(t):7.2f}  "
              f"min {min(t):7.2f}  frac {alg / m / 1e3 / 6547.5:.3f}")
