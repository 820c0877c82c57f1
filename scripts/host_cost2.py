import sys, time, ctypes
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_1404_1521_b200 as pg, synth
from paper_1404_1521_b200 import _ptr
V, d, n, h = 100_000, 64, 5, 32
m = pg.PolyglotModel(V, d, n, h, seed=42)
B = 4096
i, c = synth.batch(V, n, B, seed=1)
di, dc = torch.from_numpy(i).cuda(), torch.from_numpy(c).cuda()
loss = torch.zeros(1, device="cuda")
for k in range(5): m.train_step(di, dc, 0.1)
torch.cuda.synchronize()
N = 300
t0 = time.perf_counter()
for k in range(N): _ptr(loss, np.float32)
print("_ptr(tensor)", 1e6 * (time.perf_counter() - t0) / N, "us")
L = pg.lib()
pi, pc, pl = _ptr(di, np.int32), _ptr(dc, np.int32), _ptr(loss, np.float32)
for name, lp in (("C path, loss NULL", None), ("C path, loss device", pl)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(N): L.pg_train_step(m.handle, pi, pc, B, ctypes.c_float(0.1), lp)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "host", 1e6 * (t1 - t0) / N, "us/call; wall", 1e6 * (time.perf_counter() - t0) / N)
v = loss[0:1]
t0 = time.perf_counter()
for k in range(N): v = loss[0:1]
print("torch slice", 1e6 * (time.perf_counter() - t0) / N)
hst = torch.zeros(1).pin_memory()
t0 = time.perf_counter()
for k in range(N): hst.copy_(loss, non_blocking=True)
print("copy_ D2H nb", 1e6 * (time.perf_counter() - t0) / N)
