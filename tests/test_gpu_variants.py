"""GPU parity of the model variants of SURVEY.md §8(f) NEXT-2: the tanh
nonlinearity (PG_OPT_ACTIVATION = PG_ACT_TANH) and the summed-loss reduction (PG_OPT_REDUCTION) against the float64 oracle
with its tanh switch, on all three phase-1 paths (generic: tiny config;
register-blocked h = 32: Polyglot; tiled: h in [64, 128]), the scorer, the
DP group step and DET reproducibility.  Tolerances: SURVEY.md §8(c) T1-T5."""
import numpy as np
import pytest

import oracle
import synth
from tests._parity import assert_parity, oracle_from_gpu_params, run_both

pytestmark = pytest.mark.gpu

TINY = dict(V=1000, d=16, n=5, h=32)
POLY = dict(V=100_000, d=64, n=5, h=32)
TILED = dict(V=20_000, d=64, n=5, h=128)


@pytest.fixture(scope="module")
def pg():
    import paper_1404_1521_b200 as pg
    import torch
    assert torch.cuda.is_available()
    pg.lib()
    return pg


def make(pg, cfg, **kw):
    return pg.PolyglotModel(cfg["V"], cfg["d"], cfg["n"], cfg["h"], activation=pg.PG_ACT_TANH, **kw)


@pytest.mark.parametrize("cfg,B,steps", [(TINY, 16, 50), (POLY, 1024, 8), (TILED, 2413, 3)],
                         ids=["generic", "fast", "tiled"])
def test_tanh_parity_default_init(pg, cfg, B, steps):
    m = make(pg, cfg, seed=42)
    with oracle.activation(oracle.TANH):
        gl, rl, p0, pend, ref = run_both(m, **cfg, B=B, steps=steps)
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3)
    m.close()


@pytest.mark.parametrize("cfg", [POLY, TILED], ids=["fast", "tiled"])
def test_tanh_parity_saturated(pg, cfg):
    V, d, n, h = cfg["V"], cfg["d"], cfg["n"], cfg["h"]
    start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = make(pg, cfg, seed=1)
    with oracle.activation(oracle.TANH):
        gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=1024, steps=4, start_params=start)
        f = oracle.forward(oracle_from_gpu_params(p0, V, d, n, h), *synth.batch(V, n, 1024, seed=42, step=0))
    a = np.abs(f["a"])
    assert (a > 2).mean() > 0.02 and (a < 0.5).mean() > 0.05
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4)
    m.close()


def test_tanh_score_and_switch(pg):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    start = synth.random_params(V, d, n, h, seed=9, w1_scale=50 * 0.5 / (n * d))
    m = make(pg, POLY, seed=3)
    pg.pg_set_params(m.handle, *start[:4], b2=start[4])
    idx, _ = synth.batch(V, n, 777, seed=4)
    ref = oracle_from_gpu_params(m.get_params(), V, d, n, h)
    with oracle.activation(oracle.TANH):
        r_tanh = oracle.score(ref, idx)
    r_hard = oracle.score(ref, idx)
    s = m.score(idx)
    assert np.abs(s - r_tanh).max() <= 1e-4 * np.abs(r_tanh).max()
    assert np.abs(r_tanh - r_hard).max() > 1e-3          # the two really differ here
    pg.pg_set_option(m.handle, pg.PG_OPT_ACTIVATION, pg.PG_ACT_HARDTANH)
    s2 = m.score(idx)
    assert np.abs(s2 - r_hard).max() <= 1e-4 * np.abs(r_hard).max()
    with pytest.raises(pg.PGError) as e:
        pg.pg_set_option(m.handle, pg.PG_OPT_ACTIVATION, 7)
    assert e.value.status == pg.PG_EINVAL
    m.close()


def test_tanh_det_reproducible_fused_equals_split(pg):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    outs = []
    for fused in (True, True, False):
        m = make(pg, POLY, seed=7, fused=fused)
        ls = [m.train_step(*synth.batch(V, n, 2048, seed=3, step=t), 0.1) for t in range(3)]
        outs.append((ls, m.get_params()))
        m.close()
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        for k in range(5):
            assert np.array_equal(np.asarray(o[1][k]), np.asarray(outs[0][1][k])), k


@pytest.mark.parametrize("world", [2, 4])
def test_tanh_group_step_matches_oracle_dp(pg, world):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    models = [make(pg, POLY, seed=42) for _ in range(world)]
    p0 = models[0].get_params()
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    gl, rl = [], []
    with oracle.activation(oracle.TANH):
        for t in range(3):
            idx, corr = synth.batch(V, n, 512 * world, seed=5, step=t)
            gl.append(pg.pg_train_step_group([mm.handle for mm in models], idx, corr, 0.1))
            rl.append(oracle.train_step_dp(ref, idx, corr, 0.1, world))
    outs = [mm.get_params() for mm in models]
    for k in range(4):
        for r in range(1, world):
            assert np.array_equal(outs[0][k], outs[r][k]), (k, r)
    assert_parity(np.array(gl), np.array(rl), p0, outs[0], ref, tau_delta=1e-3)
    for mm in models:
        mm.close()


# ---------------------------------------------------------------- sum reduction (PG_OPT_REDUCTION)
@pytest.mark.parametrize("act", [0, 1], ids=["hardtanh", "tanh"])
def test_sum_reduction_parity(pg, act):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    B = 1024
    m = pg.PolyglotModel(V, d, n, h, seed=42, activation=act, reduction=pg.PG_REDUCE_SUM)
    with oracle.activation(act), oracle.reduction(oracle.SUM):
        gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=B, steps=6, lr=0.1 / B)
    assert gl[0] > 100        # a sum, not a mean
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3)
    m.close()


def test_sum_equals_mean_at_scaled_lr(pg):
    # one step of the summed loss at lr equals the mean step at lr * B; B and lr
    # powers of two so the fp32 gradient scalings are exact and the DET results
    # must agree bitwise (the loss differs by exactly B)
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    B = 2048
    idx, corr = synth.batch(V, n, B, seed=6)
    ms = pg.PolyglotModel(V, d, n, h, seed=8, reduction=pg.PG_REDUCE_SUM)
    mm = pg.PolyglotModel(V, d, n, h, seed=8)
    ls = ms.train_step(idx, corr, 2.0 ** -14)
    lm = mm.train_step(idx, corr, 2.0 ** -14 * B)
    assert ls == np.float32(lm) * B
    for a, b in zip(ms.get_params(), mm.get_params()):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    ms.close(); mm.close()


def test_tanh_atomic_scatter_parity(pg):
    """tanh with the ATOMIC embedding update (per-row red.add: one fp32
    rounding per occurrence, allowed for by c_roundings)."""
    m = make(pg, POLY, seed=42, scatter=pg.PG_SCATTER_ATOMIC)
    with oracle.activation(oracle.TANH):
        gl, rl, p0, pend, ref = run_both(m, **POLY, B=1024, steps=6)
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3, c_roundings=run_both.roundings)
    m.close()


def test_tanh_atomic_scatter_saturated(pg):
    # tanh + ATOMIC in the saturated regime: the embedding deltas pinned at tau 1e-4
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = make(pg, POLY, seed=1, scatter=pg.PG_SCATTER_ATOMIC)
    with oracle.activation(oracle.TANH):
        gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=1024, steps=4, start_params=start)
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4, c_roundings=run_both.roundings)
    m.close()


@pytest.mark.parametrize("act", [0, 1], ids=["hardtanh", "tanh"])
def test_sum_reduction_saturated(pg, act):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    B = 1024
    start = synth.random_params(V, d, n, h, seed=6, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = pg.PolyglotModel(V, d, n, h, seed=42, activation=act, reduction=pg.PG_REDUCE_SUM)
    with oracle.activation(act), oracle.reduction(oracle.SUM):
        gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=B, steps=4, lr=0.1 / B, start_params=start)
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4)
    m.close()


def test_train_step_loss_literal_form(pg):
    """pg_train_step_loss (the north-star form returning the loss): equals the
    oracle's loss; NaN plus a message naming the position on a bad index, and
    no mutation."""
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    m = make(pg, POLY, seed=3)
    idx, corr = synth.batch(V, n, 512, seed=9)
    ref = oracle_from_gpu_params(m.get_params(), V, d, n, h)
    with oracle.activation(oracle.TANH):
        lr_ = oracle.loss(ref, idx, corr)
    lg = pg.pg_train_step_loss(m.handle, idx, corr, 0.1)
    assert abs(lg - lr_) <= 1e-4 * abs(lr_)
    before = m.get_params()
    bad = idx.copy()
    bad[17, 3] = -1
    assert np.isnan(pg.pg_train_step_loss(m.handle, bad, corr, 0.1))
    msg = pg.pg_last_error()
    assert f"flat position {17 * n + 3} (value -1)" in msg, msg
    for a, b in zip(before, m.get_params()):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    m.close()
