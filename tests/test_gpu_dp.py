"""Data-parallel step on one B200: G replicas exchange their
compact records by device copies (pg_train_step_group) -- the same device code
as the NCCL path except the transport.  Checked against the oracle's G-rank
emulation (oracle.train_step_dp) and for bit-identical replicas."""
import numpy as np
import pytest

import oracle
import synth
from tests._parity import assert_parity, oracle_from_gpu_params

pytestmark = pytest.mark.gpu
POLY = dict(V=100_000, d=64, n=5, h=32)


@pytest.fixture(scope="module")
def pg():
    import paper_1404_1521_b200 as pg
    import torch
    assert torch.cuda.is_available()
    return pg


@pytest.mark.parametrize("world,B_local", [(2, 512), (4, 256), (8, 1024)])
def test_group_step_matches_oracle_dp(pg, world, B_local):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    models = [pg.PolyglotModel(V, d, n, h, seed=42) for _ in range(world)]
    p0 = models[0].get_params()
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    gl, rl = [], []
    for t in range(4):
        idx, corr = synth.batch(V, n, B_local * world, seed=5, step=t)
        gl.append(pg.pg_train_step_group([m.handle for m in models], idx, corr, 0.1))
        rl.append(oracle.train_step_dp(ref, idx, corr, 0.1, world))
    outs = [m.get_params() for m in models]
    for k in range(4):   # replicas bit-identical
        for r in range(1, world):
            assert np.array_equal(outs[0][k], outs[r][k]), (k, r)
    assert_parity(np.array(gl), np.array(rl), p0, outs[0], ref, tau_delta=2e-3)
    for m in models:
        m.close()


def test_group_equals_single_step_semantics(pg):
    # G-rank DP on a batch == one step on the whole batch, up to fp32 reordering
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    world, B_local = 4, 512
    models = [pg.PolyglotModel(V, d, n, h, seed=3) for _ in range(world)]
    single = pg.PolyglotModel(V, d, n, h, seed=3)
    idx, corr = synth.batch(V, n, B_local * world, seed=9)
    lg = pg.pg_train_step_group([m.handle for m in models], idx, corr, 0.1)
    ls = single.train_step(idx, corr, 0.1)
    assert abs(lg - ls) <= 1e-6 * abs(ls)
    a, b = models[0].get_params(), single.get_params()
    for k in range(4):
        assert np.abs(a[k] - b[k]).max() <= 1e-6 * max(1.0, np.abs(b[k]).max())
    for m in models + [single]:
        m.close()


def test_group_bad_index_on_one_rank_skips_everyone(pg):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    world, B_local = 2, 128
    models = [pg.PolyglotModel(V, d, n, h, seed=1) for _ in range(world)]
    p0 = [m.get_params() for m in models]
    idx, corr = synth.batch(V, n, B_local * world, seed=2)
    idx[B_local + 3, 2] = V + 7          # rank 1's shard
    with pytest.raises(pg.PGError) as e:
        pg.pg_train_step_group([m.handle for m in models], idx, corr, 0.1)
    assert e.value.status == pg.PG_ERANGE
    for r, m in enumerate(models):
        for a, b in zip(p0[r][:4], m.get_params()[:4]):
            assert np.array_equal(a, b)
    for m in models:
        m.close()
