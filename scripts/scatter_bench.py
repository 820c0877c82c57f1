"""Scatter-add microbench only: 1M rows into 100k x 64,
Zipf and uniform, DET and ATOMIC, L2 flushed, event-timed per call."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_1521_b200 as pg
import synth

dev = torch.device("cuda")
flush = torch.empty(128 * 1024 * 1024, device=dev)
rows, cols, N = 100_000, 64, 1_000_000
modes = [("det", 0), ("atomic", 1)] if len(sys.argv) < 2 else [(m, {"det": 0, "atomic": 1}[m]) for m in sys.argv[1:]]
for dist_name in ("zipf", "uniform"):
    I, Y = synth.scatter_inputs(rows, cols, N, dist_name, "random", seed=42)
    U = int(np.unique(I).size)
    alg = N * (4 * cols + 4) + 2 * U * 4 * cols
    Id, Yd = torch.from_numpy(I).to(dev), torch.from_numpy(Y).to(dev)
    ref = torch.zeros(rows, cols, dtype=torch.float64, device=dev).index_add_(0, Id.long(), Yd.double())
    for mode_name, mode in modes:
        W = torch.zeros(rows, cols, device=dev)
        pg.pg_scatter_add(W, Yd, Id, mode=mode)
        err = (W.double() - ref).abs().max().item()
        tms = []
        for _ in range(10):
            flush.zero_()
            if os.environ.get("SLEEP"):
                torch.cuda._sleep(int(os.environ["SLEEP"]))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            pg.pg_scatter_add_async(W, Yd, Id, mode=mode)
            b.record()
            tms.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median([a.elapsed_time(b) for a, b in tms]) * 1e3
        # back to back (no flush in between; Y is 10x larger than L2 anyway)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            pg.pg_scatter_add_async(W, Yd, Id, mode=mode)
        b.record()
        torch.cuda.synchronize()
        bb = a.elapsed_time(b) * 1e3 / 20
        print(f"{dist_name:8s} {mode_name:6s} {us:7.1f} us  {alg / us / 1e3:6.0f} GB/s  (back-to-back {bb:6.1f} us)"
              f"  max|err| vs fp64 {err:.2e}")
