"""GPU parity of pg_scatter_add (the paper's advanced-indexing op)
against the serial oracle index_add, through the C ABI."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests._parity import higham_bound

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_1404_1521_b200 as pg
    assert torch.cuda.is_available()
    return pg, torch


def gpu_scatter(env, W, Y, I, mode):
    pg, torch = env
    Wd = torch.from_numpy(W).cuda()
    pg.pg_scatter_add(Wd, torch.from_numpy(Y).cuda(), torch.from_numpy(I).cuda(), mode=mode)
    torch.cuda.synchronize()
    return Wd.cpu().numpy()


@pytest.mark.parametrize("mode", [0, 1])
def test_spec_examples(env, mode):
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        ex = json.load(f)["index_add"]
    for e in ex:
        W = np.array(e["W"], np.float32)
        Y = np.array(e["Y"], np.float32).reshape(-1, W.shape[1])
        if mode == 1:   # atomic path needs cols % 4 == 0: pad columns with zeros
            W = np.pad(W, ((0, 0), (0, 2))); Y = np.pad(Y, ((0, 0), (0, 2)))
        out = gpu_scatter(env, W, Y, np.array(e["I"], np.int32), mode)
        np.testing.assert_array_equal(out[:, :2], np.array(e["expect"], np.float32), err_msg=e["cite"])


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("dist", ["zipf", "uniform"])
def test_full_size_int_payload_bitwise(env, mode, dist):
    # BASELINE.json configs[2] at full size: 100k x 64 table, 1M rows.  Integer
    # payloads in [-8, 8]: every partial sum is an exact float32 integer
    # (|sum| <= 8 * 82712 < 2^24), so every summation order gives the serial
    # oracle's bits.
    rows, cols, n = 100_000, 64, 1_000_000
    I, Y = synth.scatter_inputs(rows, cols, n, dist, "int", seed=3)
    W0 = ((synth.uniform_ids(17, rows * cols, 5, 99, 0) - 8).astype(np.float32)).reshape(rows, cols)
    ref = oracle.index_add(W0.copy(), Y, I)
    out = gpu_scatter(env, W0.copy(), Y, I, mode)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("mode", [0, 1])
def test_full_size_random_payload(env, mode):
    rows, cols, n = 100_000, 64, 1_000_000
    I, Y = synth.scatter_inputs(rows, cols, n, "zipf", "random", seed=4)
    W0 = np.zeros((rows, cols), np.float32)
    ref = oracle.index_add(W0.astype(np.float64), Y.astype(np.float64), I)
    out = gpu_scatter(env, W0.copy(), Y, I, mode)
    err = np.abs(out - ref)
    # float32 reordering error, relative to each row's infinity norm (the T2
    # reading of "1e-4 relative" applied per embedding row) ...
    scale = np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1e-30)
    assert (err / scale).max() <= 1e-4, (err / scale).max()
    # ... and within the worst-case fp32 summation bound of each element
    assert (err <= higham_bound(W0, Y, I)).all()


def test_det_bitwise_run_to_run(env):
    rows, cols, n = 100_000, 64, 1_000_000
    I, Y = synth.scatter_inputs(rows, cols, n, "zipf", "random", seed=6)
    W0 = np.zeros((rows, cols), np.float32)
    a = gpu_scatter(env, W0.copy(), Y, I, 0)
    b = gpu_scatter(env, W0.copy(), Y, I, 0)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("cols", [4, 16, 32, 64, 128])
def test_fuzz_small(env, mode, cols):
    # fuzz over rows <= 100, updates <= 500, duplicate rates 0 / 0.5 / 1
    rng = np.random.default_rng(cols * 10 + mode)
    for case in range(20):
        rows = int(rng.integers(1, 101))
        n = int(rng.integers(0, 501))
        dup = [0.0, 0.5, 1.0][case % 3]
        if dup == 1.0:
            I = np.full(n, rng.integers(0, rows), np.int32)
        elif dup == 0.0:
            I = rng.permutation(max(rows, n))[:n].astype(np.int32) % rows
        else:
            I = rng.integers(0, max(1, rows // 2), n).astype(np.int32)
        Y = rng.standard_normal((n, cols)).astype(np.float32)
        W0 = rng.standard_normal((rows, cols)).astype(np.float32)
        ref = oracle.index_add(W0.astype(np.float64), Y.astype(np.float64), I)
        if n == 0:
            continue
        out = gpu_scatter(env, W0.copy(), Y, I, mode)
        # any fp32 summation order of a row's m terms is within
        # gamma_m * sum|terms| of the exact sum (Higham); the oracle is fp64
        assert (np.abs(out - ref) <= higham_bound(W0, Y, I)).all()


def test_out_of_range_leaves_w_unchanged(env):
    pg, torch = env
    rows, cols, n = 1000, 64, 5000
    I, Y = synth.scatter_inputs(rows, cols, n, "uniform", "random")
    I[1234] = rows
    for mode in (0, 1):
        W = torch.ones(rows, cols, device="cuda")
        with pytest.raises(pg.PGError) as e:
            pg.pg_scatter_add(W, torch.from_numpy(Y).cuda(), torch.from_numpy(I).cuda(), mode=mode)
        assert e.value.status == pg.PG_ERANGE and "position 1234" in str(e.value)
        assert bool((W == 1).all())


def test_empty_is_noop(env):
    pg, torch = env
    W = torch.ones(10, 64, device="cuda")
    pg.pg_scatter_add(W, torch.zeros(0, 64, device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert bool((W == 1).all())


def test_atomic_error_slots_alternate(env):
    """ATOMIC reports through two status slots used on alternate calls (no
    per-call reset): a bad call, then good calls, then a bad one must each
    report their own outcome, and only the good ones change W."""
    pg, torch = env
    rows, cols, n = 500, 64, 3000
    I, Y = synth.scatter_inputs(rows, cols, n, "zipf", "int", seed=5)
    Yd = torch.from_numpy(Y).cuda()
    bad = I.copy()
    bad[17] = -3
    W = torch.zeros(rows, cols, device="cuda")
    ref = np.zeros((rows, cols), np.float64)
    for k, ok in enumerate([False, True, True, False, False, True]):
        Id = torch.from_numpy(I if ok else bad).cuda()
        if ok:
            pg.pg_scatter_add(W, Yd, Id, mode=pg.PG_SCATTER_ATOMIC)
            ref = oracle.index_add(ref, Y.astype(np.float64), I)
        else:
            with pytest.raises(pg.PGError) as e:
                pg.pg_scatter_add(W, Yd, Id, mode=pg.PG_SCATTER_ATOMIC)
            assert e.value.status == pg.PG_ERANGE and "position 17" in str(e.value), k
        assert np.array_equal(W.cpu().numpy(), ref.astype(np.float32)), k


def test_atomic_async_err_flag(env):
    pg, torch = env
    rows, cols, n = 200, 16, 1000
    I, Y = synth.scatter_inputs(rows, cols, n, "uniform", "int", seed=6)
    I[999] = rows
    W = torch.zeros(rows, cols, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for k in range(3):   # both status slots
        pg.pg_scatter_add_async(W, torch.from_numpy(Y).cuda(), torch.from_numpy(I).cuda(),
                                mode=pg.PG_SCATTER_ATOMIC, err_flag=flag)
        torch.cuda.synchronize()
        assert int(flag.item()) == 1 and bool((W == 0).all()), k
        flag.zero_()


def test_unaligned_rejected(env):
    pg, torch = env
    buf = torch.zeros(10 * 64 + 1, device="cuda")
    W = buf[1:].view(10, 64)   # 4-byte aligned only
    with pytest.raises(pg.PGError) as e:
        pg.pg_scatter_add(W, torch.ones(3, 64, device="cuda"), torch.zeros(3, dtype=torch.int32, device="cuda"),
                          mode=pg.PG_SCATTER_ATOMIC)
    assert e.value.status == pg.PG_EINVAL


@pytest.mark.parametrize("cols", [4, 12, 64, 128])
def test_atomic_hot_rows_int_payload_bitwise(env, cols):
    """Heavily repeated rows (every tier of the ATOMIC hot set: a 30 % row,
    a Zipf head, single-use rows) with integer payloads: every summation order
    is exact, so ATOMIC must equal the serial oracle bitwise at every width."""
    rng = np.random.default_rng(cols)
    rows, n = 5000, 200_000
    I = np.where(rng.random(n) < 0.3, 7, rng.zipf(1.3, n) % rows).astype(np.int32)
    Y = rng.integers(-8, 9, (n, cols)).astype(np.float32)
    ref = oracle.index_add(np.zeros((rows, cols), np.float32), Y, I)
    assert np.array_equal(gpu_scatter(env, np.zeros((rows, cols), np.float32), Y, I, 1), ref)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("cols", [1, 5, 30])
def test_odd_widths_int_payload_bitwise(env, mode, cols):
    """Widths that are not a multiple of 4 (scalar paths) with integer payloads
    and Zipf-repeated rows: bitwise equal to the serial oracle."""
    rng = np.random.default_rng(100 + cols)
    rows, n = 3000, 50_000
    I = (rng.zipf(1.2, n) % rows).astype(np.int32)
    Y = rng.integers(-8, 9, (n, cols)).astype(np.float32)
    ref = oracle.index_add(np.zeros((rows, cols), np.float32), Y, I)
    assert np.array_equal(gpu_scatter(env, np.zeros((rows, cols), np.float32), Y, I, mode), ref)


def test_det_multi_launch_sort_above_one_tile_per_sm(env):
    """n above 148 x 8192 = 1.21M entries: the DET radix sort leaves the one-
    launch cooperative form for the multi-launch upsweep / scan / downsweep
    pipeline.  Integer payloads: bitwise equal to the serial oracle, and run to
    run."""
    rows, cols, n = 100_000, 64, 1_600_000
    I, Y = synth.scatter_inputs(rows, cols, n, "zipf", "int", seed=8)
    ref = oracle.index_add(np.zeros((rows, cols), np.float32), Y, I)
    a = gpu_scatter(env, np.zeros((rows, cols), np.float32), Y, I, 0)
    assert np.array_equal(a, ref)
    I2, Y2 = synth.scatter_inputs(rows, cols, n, "uniform", "random", seed=9)
    b1 = gpu_scatter(env, np.zeros((rows, cols), np.float32), Y2, I2, 0)
    b2 = gpu_scatter(env, np.zeros((rows, cols), np.float32), Y2, I2, 0)
    assert np.array_equal(b1, b2)


@pytest.mark.parametrize("cols", [132, 256])
def test_atomic_vector_fallback_wide_rows(env, cols):
    """ATOMIC with cols % 4 == 0 but cols > 128 takes the plain vector
    red.global.add.v4.f32 kernel (sc_atomic) instead of the hot-set kernel:
    integer payloads with Zipf-repeated rows, bitwise equal to the oracle."""
    rng = np.random.default_rng(cols)
    rows, n = 4000, 60_000
    I = (rng.zipf(1.2, n) % rows).astype(np.int32)
    Y = rng.integers(-8, 9, (n, cols)).astype(np.float32)
    ref = oracle.index_add(np.zeros((rows, cols), np.float32), Y, I)
    assert np.array_equal(gpu_scatter(env, np.zeros((rows, cols), np.float32), Y, I, 1), ref)
