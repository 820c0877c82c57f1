"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): the fused step (tiny + Polyglot shapes,
DET and ATOMIC, fused and split), the tiled path, both scatter-add modes, and
the data-parallel publish / merge (PEER emulation, G = 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_1521_b200 as pg
import synth

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "step"):
    for (V, d, n, h, B) in ((1000, 16, 5, 32, 16), (100_000, 64, 5, 32, 1024), (20_000, 64, 5, 128, 300)):
        for scatter in (0, 1):
            for fused in (True, False):
                m = pg.PolyglotModel(V, d, n, h, seed=1, scatter=scatter, fused=fused)
                for t in range(2):
                    idx, corr = synth.batch(V, n, B, seed=2, step=t)
                    m.train_step(idx, corr, 0.1)
                m.close()
if which in ("all", "scatter"):
    for mode in (0, 1):
        for dist in ("zipf", "uniform"):
            I, Y = synth.scatter_inputs(5000, 64, 20_000, dist, "random", seed=3)
            W = torch.zeros(5000, 64, device="cuda")
            pg.pg_scatter_add(W, torch.from_numpy(Y).cuda(), torch.from_numpy(I).cuda(), mode=mode)
if which in ("all", "dp"):
    V, d, n, h = 100_000, 64, 5, 32
    ms = [pg.PolyglotModel(V, d, n, h, seed=1, exchange=pg.PG_EXCHANGE_PEER) for _ in range(2)]
    for t in range(2):
        idx, corr = synth.batch(V, n, 512, seed=4, step=t)
        pg.pg_train_step_group([m.handle for m in ms], idx, corr, 0.1)
    for m in ms:
        m.close()
torch.cuda.synchronize()
print("sanitize run ok", which)
