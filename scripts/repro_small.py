import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1404_1521_b200 as pg
cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
V, d, n, h, B = (1000, 16, 5, 32, 16) if cfg == "tiny" else (100000, 64, 5, 32, int(sys.argv[2]) if len(sys.argv) > 2 else 256)
m = pg.PolyglotModel(V, d, n, h, fused=("split" not in sys.argv))
for t in range(2):
    idx, corr = synth.batch(V, n, B, seed=1, step=t)
    print(m.train_step(idx, corr, 0.1))
