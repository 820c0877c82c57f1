"""Host-side cost per pg_train_step call (device / pinned inputs, device loss) against the
GPU step time, and the bare ctypes call floor."""
import sys, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1404_1521_b200 as pg, synth
V, d, n, h = 100_000, 64, 5, 32
m = pg.PolyglotModel(V, d, n, h, seed=42)
B = 4096
bs = [synth.batch(V, n, B, seed=1, step=t) for t in range(8)]
di = [torch.from_numpy(i).cuda() for i, _ in bs]; dc = [torch.from_numpy(c).cuda() for _, c in bs]
pi = [torch.from_numpy(i).pin_memory() for i, _ in bs]; pc = [torch.from_numpy(c).pin_memory() for _, c in bs]
loss = torch.zeros(1, device="cuda")
for k in range(5): m.train_step(di[0], dc[0], 0.1)
torch.cuda.synchronize()
for name, I, Cc, lo in (("device in, no loss", di, dc, None), ("device in, dev loss", di, dc, loss), ("pinned in, dev loss", pi, pc, loss)):
    N = 200
    t0 = time.perf_counter()
    for k in range(N): m.train_step(I[k % 8], Cc[k % 8], 0.1, loss_out=lo)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:22s} host {1e6*(t1-t0)/N:6.1f} us/call, wall {1e6*(t2-t0)/N:6.1f} us/step")
# ctypes-only floor
t0 = time.perf_counter()
for k in range(2000): pg.lib().pg_abi_version()
print("ctypes call", 1e6*(time.perf_counter()-t0)/2000, "us")
