"""Quick step timing: L2-flushed and back-to-back us/step for a few batch sizes (Polyglot shape)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1404_1521_b200 as pg
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="16,1024,2048,4096,8192")
ap.add_argument("--atomic", action="store_true")
ap.add_argument("--large", action="store_true")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
V, d, n, h = (1_000_000, 128, 5, 128) if a.large else (100_000, 64, 5, 32)
dev = torch.device("cuda")
stream = torch.cuda.Stream()
m = pg.PolyglotModel(V, d, n, h, seed=42, stream=stream, scatter=1 if a.atomic else 0)
flush = torch.empty(128 * 1024 * 1024, device=dev)
for B in [int(x) for x in a.batches.split(",")]:
    m.reserve(B)
    bs = [synth.batch(V, n, B, seed=7, step=t) for t in range(a.reps)]
    di = [torch.from_numpy(i).to(dev) for i, _ in bs]
    dc = [torch.from_numpy(c).to(dev) for _, c in bs]
    with torch.cuda.stream(stream):
        for t in range(3):
            m.train_step(di[t], dc[t], 0.1, loss_out=None)
        torch.cuda.synchronize()
        ev = []
        for t in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            m.train_step(di[t], dc[t], 0.1, loss_out=None)
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        fl = [x.elapsed_time(y) * 1e3 for x, y in ev]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(a.reps):
            m.train_step(di[t], dc[t], 0.1, loss_out=None)
        e1.record(stream)
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) * 1e3 / a.reps
    print(f"B={B:6d} flushed {statistics.median(fl):7.2f} us (mean {statistics.mean(fl):7.2f})  back-to-back {b2b:7.2f} us"
          f"  -> {B / statistics.mean(fl) * 1e6 / 1e6:7.1f} M ex/s flushed", flush=True)
m.sync()
