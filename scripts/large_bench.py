"""Step time at the large config (BASELINE.json configs[3]: V 1M, d 128, n 5,
h 128) on one GPU, L2 flushed, for a few per-GPU batches."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1404_1521_b200 as pg
import synth

V, d, n, h = 1_000_000, 128, 5, 128
m = pg.PolyglotModel(V, d, n, h, seed=42)
fl = torch.empty(128 * 1024 * 1024, device="cuda")
for B in (512, 4096):
    bs = [synth.batch(V, n, B, seed=3, step=t) for t in range(6)]
    di = [torch.from_numpy(i).cuda() for i, _ in bs]
    dc = [torch.from_numpy(c).cuda() for _, c in bs]
    for t in range(2):
        m.train_step(di[t], dc[t], 0.1, loss_out=None)
    torch.cuda.synchronize()
    tms = []
    for t in range(2, 6):
        fl.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.train_step(di[t], dc[t], 0.1, loss_out=None)
        b.record()
        tms.append((a, b))
    torch.cuda.synchronize()
    us = statistics.median([a.elapsed_time(b) for a, b in tms]) * 1e3
    fma = (n * d * h + d * h) + ((n + 1) * d * h) + ((n + 1) * d * h)   # forward (shared context), G rows, dW1
    print(f"large B={B}: {us:8.1f} us/step  {B / us * 1e6:12.0f} ex/s  {2 * fma * B / us / 1e6:6.2f} TFLOP/s")
