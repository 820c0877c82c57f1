"""Large config (V 1M, d 128, n 5, h 128) step time across per-GPU batches (L2 flushed)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1404_1521_b200 as pg
V, d, n, h = 1_000_000, 128, 5, 128
s = torch.cuda.Stream()
m = pg.PolyglotModel(V, d, n, h, stream=s)
fl = torch.empty(128 * 1024 * 1024, device="cuda")
for B in (148, 512, 600, 1024, 1184, 2048, 4096):
    m.reserve(B)
    bs = [synth.batch(V, n, B, seed=1, step=t) for t in range(8)]
    di = [torch.from_numpy(i).cuda() for i, _ in bs]; dc = [torch.from_numpy(c).cuda() for _, c in bs]
    with torch.cuda.stream(s):
        for t in range(3): m.train_step(di[t], dc[t], 0.1, loss_out=None)
        ev = []
        for t in range(8):
            fl.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); m.train_step(di[t], dc[t], 0.1, loss_out=None); b.record(s); ev.append((a, b))
    torch.cuda.synchronize()
    us = 1e3 * statistics.median([a.elapsed_time(b) for a, b in ev])
    print(f"B={B:5d}  {us:7.1f} us/step  {B / us:6.2f} M ex/s")
