import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle, paper_1404_1521_b200 as pg
from tests._parity import oracle_from_gpu_params
V, d, n, h = 100000, 64, 5, 32
for B in (150, 256, 1024, 4096):
    rng = np.random.default_rng(0)
    idx = (rng.integers(0, V // 148, size=(B, n)) * 148).astype(np.int32)
    corr = (rng.integers(0, V // 148, size=B) * 148).astype(np.int32)
    m = pg.PolyglotModel(V, d, n, h, seed=42)
    p0 = m.get_params()
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    lg = m.train_step(idx, corr, 0.1); lr = oracle.train_step(ref, idx, corr, 0.1)
    C = m.get_params()[0]
    dg = C.astype(np.float64) - p0[0]; dr = ref.C - p0[0]
    err = np.abs(dg - dr); r = np.unravel_index(err.argmax(), err.shape)
    rows_bad = np.where(err.max(1) > 1e-3 * np.abs(dr).max())[0]
    print(B, "loss", lg, lr, "max err", err.max(), "max dref", np.abs(dr).max(), "at", r, "bad rows", len(rows_bad), rows_bad[:8], "ratio", (dg[r[0]] / dr[r[0]])[:4])
    m.close()
