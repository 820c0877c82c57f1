"""Step time: eager launches vs a captured CUDA graph (warm L2), B from argv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1404_1521_b200 as pg
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
fused = "split" not in sys.argv
V, d, n, h = 100_000, 64, 5, 32
s = torch.cuda.Stream()
m = pg.PolyglotModel(V, d, n, h, stream=s, fused=fused)
m.reserve(B)
K = 50
bs = [synth.batch(V, n, B, seed=1, step=t) for t in range(K)]
di = [torch.from_numpy(i).cuda() for i, _ in bs]; dc = [torch.from_numpy(c).cuda() for _, c in bs]
loss = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
with torch.cuda.stream(s):
    for t in range(5): m.train_step(di[t], dc[t], 0.1, loss_out=loss)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for t in range(K): m.train_step(di[t], dc[t], 0.1, loss_out=loss)
    e1.record(s)
torch.cuda.synchronize()
print(f"B={B} fused={fused} eager back-to-back: {e0.elapsed_time(e1)/K*1e3:.1f} us/step")
try:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(K): m.train_step(di[t], dc[t], 0.1, loss_out=loss)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay(); torch.cuda.synchronize()
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    print(f"B={B} fused={fused} graph of {K} steps: {e0.elapsed_time(e1)/K*1e3:.1f} us/step")
except Exception as ex:
    print("graph capture failed:", repr(ex)[:300])
