"""GPU parity of the TILED phase-1 path (h % 32 == 0, 64 <= h <= 128 -- the
large config's shape family) against the float64 oracle: several shapes,
ragged and multi-chunk batches, the saturated regime, DET reproducibility,
fused == split, the bad-index gate, set_params (which refreshes the W1^T
mirror the path reads) and the data-parallel group step.
Tolerances: SURVEY.md §8(c) T1-T5."""
import numpy as np
import pytest

import oracle
import synth
from tests._parity import assert_parity, oracle_from_gpu_params, run_both

pytestmark = pytest.mark.gpu

SHAPES = [dict(V=5000, d=32, n=5, h=64), dict(V=20_000, d=64, n=3, h=96), dict(V=50_000, d=128, n=5, h=128)]


@pytest.fixture(scope="module")
def pg():
    import paper_1404_1521_b200 as pg
    import torch
    assert torch.cuda.is_available()
    pg.lib()
    return pg


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: f"d{c['d']}n{c['n']}h{c['h']}")
@pytest.mark.parametrize("B", [5, 300, 580, 1000, 2400 + 13])   # 4-, 4-, 4-, 8- and 16-example chunks
def test_tiled_parity(pg, cfg, B):
    # B = 580: the dW1 GEMM's 5 passes of 128 examples refill its 4-buffer TMA
    # ring mid-tile; B = 2413 > 148 * 16: several 16-example chunks per CTA
    # (record RMW path)
    m = pg.PolyglotModel(cfg["V"], cfg["d"], cfg["n"], cfg["h"], seed=11)
    gl, rl, p0, pend, ref = run_both(m, **cfg, B=B, steps=3, kind="iid" if B < 100 else "sliding")
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3)
    m.close()


def test_tiled_saturated_regime(pg):
    V, d, n, h = 20_000, 64, 5, 128
    start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = pg.PolyglotModel(V, d, n, h, seed=1)
    gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=1024, steps=4, start_params=start)
    f = oracle.forward(oracle_from_gpu_params(p0, V, d, n, h), *synth.batch(V, n, 1024, seed=42, step=0))
    a = np.abs(np.concatenate([f["a"].ravel(), f["a_corr"].ravel()]))
    assert (a > 1).mean() > 0.2 and (a < 1).mean() > 0.2   # both hardtanh regions exercised
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4)
    m.close()


def test_tiled_det_reproducible_and_fused_equals_split(pg):
    V, d, n, h = 20_000, 64, 5, 96
    outs = []
    for fused in (True, True, False):
        m = pg.PolyglotModel(V, d, n, h, seed=4, fused=fused)
        for t in range(3):
            idx, corr = synth.batch(V, n, 3000, seed=8, step=t)
            m.train_step(idx, corr, 0.1)
        outs.append(m.get_params())
        m.close()
    for k in range(4):
        assert np.array_equal(outs[0][k], outs[1][k]), "T5: det run-to-run"
        assert np.array_equal(outs[0][k], outs[2][k]), "fused vs split"


def test_tiled_bad_index_and_set_params(pg):
    V, d, n, h = 5000, 32, 5, 64
    m = pg.PolyglotModel(V, d, n, h, seed=2)
    idx, corr = synth.batch(V, n, 500, seed=3)
    p0 = m.get_params()
    bad = idx.copy(); bad[100, 1] = V + 7
    with pytest.raises(pg.PGError) as e:
        m.train_step(bad, corr, 0.1)
    assert e.value.status == pg.PG_ERANGE
    for a, b in zip(p0[:4], m.get_params()[:4]):
        assert np.array_equal(a, b)
    # new W1 through the ABI: the step must use it (the W1^T mirror is refreshed)
    start = synth.random_params(V, d, n, h, seed=9)
    m.set_params(*start)
    gl, rl, q0, qend, ref = run_both(m, V, d, n, h, B=500, steps=2)
    assert np.array_equal(q0[1], start[1].astype(np.float32))
    assert_parity(gl, rl, q0, qend, ref, tau_delta=1e-3)
    m.close()


@pytest.mark.parametrize("world,sat", [(2, False), (4, False), (4, True)])
def test_tiled_group_step_matches_oracle_dp(pg, world, sat):
    V, d, n, h = 20_000, 64, 5, 128
    models = [pg.PolyglotModel(V, d, n, h, seed=42) for _ in range(world)]
    if sat:
        start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
        for mm in models:
            mm.set_params(*start[:4], b2=start[4])
    p0 = models[0].get_params()
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    gl, rl = [], []
    for t in range(3):
        idx, corr = synth.batch(V, n, 400 * world, seed=5, step=t)
        gl.append(pg.pg_train_step_group([mm.handle for mm in models], idx, corr, 0.1))
        rl.append(oracle.train_step_dp(ref, idx, corr, 0.1, world))
    outs = [mm.get_params() for mm in models]
    for k in range(4):
        for r in range(1, world):
            assert np.array_equal(outs[0][k], outs[r][k]), (k, r)
    assert_parity(np.array(gl), np.array(rl), p0, outs[0], ref, tau_delta=1e-4 if sat else 1e-3)
    for mm in models:
        mm.close()
