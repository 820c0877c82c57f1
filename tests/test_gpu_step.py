"""GPU parity of the fused SGD step (libpg, sm_100a) against the float64 oracle.

All calls go through the C ABI (paper_1404_1521_b200 ctypes binding).
Tolerances: SURVEY.md §8(c) T1-T5, restated in DESIGN.md.
"""
import numpy as np
import pytest

import oracle
import synth
from tests._parity import assert_parity, oracle_from_gpu_params, rel_inf, run_both

pytestmark = pytest.mark.gpu

TINY = dict(V=1000, d=16, n=5, h=32)
POLY = dict(V=100_000, d=64, n=5, h=32)


@pytest.fixture(scope="module")
def pg():
    import paper_1404_1521_b200 as pg
    import torch
    assert torch.cuda.is_available()
    pg.lib()
    return pg


def make(pg, cfg, seed=42, scatter=0, fused=True):
    return pg.PolyglotModel(cfg["V"], cfg["d"], cfg["n"], cfg["h"], seed=seed, scatter=scatter,
                            fused=fused)


def test_init_matches_oracle_init_bitwise(pg):
    for cfg in (TINY, POLY):
        m = make(pg, cfg, seed=1234)
        C, W1, b1, w2, b2 = m.get_params()
        ref = oracle.Params.init(cfg["V"], cfg["d"], cfg["n"], cfg["h"], 1234)
        np.testing.assert_array_equal(C.astype(np.float64), ref.C)
        np.testing.assert_array_equal(W1.astype(np.float64), ref.W1)
        np.testing.assert_array_equal(w2.astype(np.float64), ref.w2)
        assert not b1.any() and b2 == 0.0
        m.close()


@pytest.mark.parametrize("scatter", [0, 1])
def test_tiny_100_steps(pg, scatter):
    # BASELINE.json configs[0]: tiny, batch 16, 100 SGD steps (generic kernel path)
    m = make(pg, TINY, scatter=scatter)
    gl, rl, p0, pend, ref = run_both(m, **TINY, B=16, steps=100)
    rep = assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3,
                        c_roundings=run_both.roundings if scatter else None)
    print("tiny", scatter, rep)
    m.close()


@pytest.mark.parametrize("scatter", [0, 1])
def test_polyglot_b1024_default_init(pg, scatter):
    m = make(pg, POLY, scatter=scatter)
    gl, rl, p0, pend, ref = run_both(m, **POLY, B=1024, steps=20)
    rep = assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3,
                        c_roundings=run_both.roundings if scatter else None)
    print("poly", scatter, rep)
    m.close()


@pytest.mark.parametrize("scatter", [0, 1])
def test_polyglot_saturated_regime(pg, scatter):
    # W1, w2 scaled x200 so units saturate and margins go negative (T3: tau 1e-4)
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = make(pg, POLY, scatter=scatter)
    gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=1024, steps=20, start_params=start)
    f = oracle.forward(oracle_from_gpu_params(p0, V, d, n, h), *synth.batch(V, n, 1024, seed=42, step=0))
    assert (np.abs(f["a"]) > 1).mean() > 0.2          # really saturated
    rep = assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4,
                        c_roundings=run_both.roundings if scatter else None)
    print("sat", scatter, rep)
    m.close()


@pytest.mark.parametrize("B", [1, 7, 149, 1000, 4096 + 37, 9000])
def test_ragged_batches(pg, B):
    # ragged tails, fewer examples than SMs, and several chunks per CTA (B > 148*32)
    m = make(pg, POLY)
    gl, rl, p0, pend, ref = run_both(m, **POLY, B=B, steps=3, kind="iid")
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3)
    m.close()


SAT = lambda V, d, n, h, seed=5: synth.random_params(V, d, n, h, seed=seed, w1_scale=200 * 0.5 / (n * d),
                                                      w2_scale=200 * 0.5 / h)


@pytest.mark.parametrize("scatter", [0, 1])
@pytest.mark.parametrize("B", [1, 7, 149, 1000, 4096 + 37, 9000])
def test_ragged_batches_saturated(pg, B, scatter):
    # the ragged shapes in the saturated regime: embedding updates far above the
    # fp32 storage floor, so T3 pins every tensor's delta at tau = 1e-4
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    m = make(pg, POLY, scatter=scatter)
    gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=B, steps=3, kind="iid", start_params=SAT(V, d, n, h))
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4, c_roundings=run_both.roundings if scatter else None)
    m.close()


def test_det_bitwise_reproducible_and_fused_equals_split(pg):
    outs = []
    for fused in (True, True, False):
        m = make(pg, POLY, fused=fused)
        for t in range(5):
            idx, corr = synth.batch(POLY["V"], POLY["n"], 2048, seed=7, step=t)
            m.train_step(idx, corr, 0.1)
        outs.append(m.get_params())
        m.close()
    for k in range(4):
        assert np.array_equal(outs[0][k], outs[1][k]), "T5: det run-to-run"
        assert np.array_equal(outs[0][k], outs[2][k]), "fused vs split"


def test_bad_index_no_mutation(pg):
    m = make(pg, POLY)
    p0 = m.get_params()
    idx, corr = synth.batch(POLY["V"], POLY["n"], 256, seed=1)
    bad = idx.copy(); bad[17, 3] = POLY["V"]
    with pytest.raises(pg.PGError) as e:
        m.train_step(bad, corr, 0.1)
    assert e.value.status == pg.PG_ERANGE
    assert f"position {17 * 5 + 3} (value {POLY['V']})" in str(e.value)
    badc = corr.copy(); badc[3] = -5
    with pytest.raises(pg.PGError) as e:
        m.train_step(idx, badc, 0.1)
    assert f"position {256 * 5 + 3} (value -5)" in str(e.value)
    p1 = m.get_params()
    for a, b in zip(p0[:4], p1[:4]):
        assert np.array_equal(a, b)
    # the model keeps working afterwards
    loss = m.train_step(idx, corr, 0.1)
    assert np.isfinite(loss)
    m.close()


def test_host_checked_errors(pg):
    m = make(pg, TINY)
    idx, corr = synth.batch(TINY["V"], TINY["n"], 4, seed=1)
    for lr in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(pg.PGError) as e:
            m.train_step(idx, corr, lr)
        assert e.value.status == pg.PG_EINVAL
    with pytest.raises(pg.PGError) as e:
        m.train_step(idx[:0], corr[:0], 0.1)
    assert e.value.status == pg.PG_EINVAL
    m.close()


def test_zero_params_fixed_point(pg):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    m = make(pg, POLY)
    m.set_params(np.zeros((V, d)), np.zeros((n * d, h)), np.zeros(h), np.zeros(h), 0.0)
    for t in range(3):
        idx, corr = synth.batch(V, n, 512, seed=3, step=t)
        assert m.train_step(idx, corr, 0.1) == 1.0
    for a in m.get_params()[:4]:
        assert not a.any()
    m.close()


def test_locality_untouched_rows_bit_identical(pg):
    V, n = POLY["V"], POLY["n"]
    m = make(pg, POLY)
    C0 = m.get_params()[0]
    idx, corr = synth.batch(V, n, 1024, seed=9)
    m.train_step(idx, corr, 0.1)
    C1 = m.get_params()[0]
    touched = np.zeros(V, bool); touched[idx.ravel()] = True; touched[corr] = True
    assert np.array_equal(C1[~touched], C0[~touched])
    assert (C1[touched] != C0[touched]).any()
    m.close()


def test_score_matches_oracle(pg):
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    m = make(pg, POLY)
    p = m.get_params()
    idx, _ = synth.batch(V, n, 777, seed=4)
    s = m.score(idx)
    r = oracle.score(oracle_from_gpu_params(p, V, d, n, h), idx)
    assert np.abs(s - r).max() <= 1e-4 * np.abs(r).max()
    bad = idx.copy(); bad[5, 0] = V + 3
    with pytest.raises(pg.PGError) as e:
        m.score(bad)
    assert e.value.status == pg.PG_ERANGE
    m.close()


def test_device_pointers_async_loss(pg):
    import torch
    V, n = POLY["V"], POLY["n"]
    a, b = make(pg, POLY), make(pg, POLY)
    dl = torch.zeros(1, dtype=torch.float32, device="cuda")
    for t in range(3):
        idx, corr = synth.batch(V, n, 1024, seed=11, step=t)
        la = a.train_step(idx, corr, 0.1)
        b.train_step(torch.from_numpy(idx).cuda(), torch.from_numpy(corr).cuda(), 0.1, loss_out=dl)
        torch.cuda.synchronize()
        assert dl.item() == la
    b.sync()
    for x, y in zip(a.get_params()[:4], b.get_params()[:4]):
        assert np.array_equal(x, y)
    a.close(); b.close()


def test_large_shape_generic_path(pg):
    # BASELINE.json configs[4] shape (V 1M, d 128, h 128) on one GPU, small batch
    V, d, n, h = 1_000_000, 128, 5, 128
    m = pg.PolyglotModel(V, d, n, h, seed=3)
    gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=512, steps=3)
    assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3)
    m.close()


def test_large_shape_saturated(pg):
    # the large config's shape at its per-GPU batch (4096 / 8 = 512) and at 4096,
    # saturated regime: T3 at tau = 1e-4 pins the embedding update
    V, d, n, h = 1_000_000, 128, 5, 128
    start = SAT(V, d, n, h, seed=7)
    for B, steps in ((512, 3), (4096, 2)):
        m = pg.PolyglotModel(V, d, n, h, seed=3)
        gl, rl, p0, pend, ref = run_both(m, V, d, n, h, B=B, steps=steps, start_params=start)
        assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-4)
        m.close()


def test_owner_overflow_sorted_fallback(pg):
    # every row id is a multiple of 148 -> all gradient rows belong to owner 0,
    # whose entry count exceeds the hash fast path (sorted fallback, several windows)
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    B = 4096
    rng = np.random.default_rng(0)
    idx = (rng.integers(0, V // 148, size=(B, n)) * 148).astype(np.int32)
    corr = (rng.integers(0, V // 148, size=B) * 148).astype(np.int32)
    # saturated regime: embedding updates far above the fp32 storage floor
    start = synth.random_params(V, d, n, h, seed=5, w1_scale=200 * 0.5 / (n * d), w2_scale=200 * 0.5 / h)
    m = make(pg, POLY)
    m.set_params(*start[:4], b2=start[4])
    p0 = m.get_params()
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    gl = [m.train_step(idx, corr, 0.1)]
    rl = [oracle.train_step(ref, idx, corr, 0.1)]
    assert_parity(np.array(gl), np.array(rl), p0, m.get_params(), ref, tau_delta=1e-4)
    m.close()


@pytest.mark.timeout(300)
def test_one_model_many_batch_sizes(pg):
    # the grid size P = min(#SMs, B) changes with the batch; the fused kernel's
    # grid barrier must stay consistent across launches of different grids
    m = make(pg, POLY)
    for B in (4096, 16, 4096, 7, 149, 100, 4096, 1, 2048):
        idx, corr = synth.batch(POLY["V"], POLY["n"], B, seed=3, step=B)
        loss = m.train_step(idx, corr, 0.1)
        assert np.isfinite(loss)
    m.close()


def test_async_host_inputs_pipeline_equals_device_inputs(pg):
    # host (pinned and pageable) inputs are staged on a copy stream into two
    # alternating device slots; many steps in flight must give exactly the
    # parameters of the same steps fed from device memory
    import torch
    batches = [synth.batch(POLY["V"], POLY["n"], 1024, seed=21, step=t) for t in range(12)]
    a = make(pg, POLY, seed=5)
    b = make(pg, POLY, seed=5)
    loss_a = torch.zeros(12, device="cuda")
    for t, (i, c) in enumerate(batches):
        hi = torch.from_numpy(i).pin_memory() if t % 2 == 0 else i      # pinned / pageable
        hc = torch.from_numpy(c).pin_memory() if t % 2 == 0 else c
        a.train_step(hi, hc, 0.1, loss_out=loss_a[t:t + 1])
    a.sync()
    lb = [b.train_step(torch.from_numpy(i).cuda(), torch.from_numpy(c).cuda(), 0.1) for i, c in batches]
    assert np.array_equal(loss_a.cpu().numpy(), np.array(lb, np.float32))
    for x, y in zip(a.get_params()[:4], b.get_params()[:4]):
        assert np.array_equal(x, y)
    a.close(); b.close()


def test_pinned_host_loss_is_written_asynchronously(pg):
    # a page-locked host loss_out makes the call asynchronous: the step kernel
    # stores the loss through the buffer's device mapping (include/pg.h); after
    # a sync the values equal the blocking call's, and the parameters match
    import torch
    batches = [synth.batch(POLY["V"], POLY["n"], 1024, seed=23, step=t) for t in range(6)]
    a = make(pg, POLY, seed=9)
    b = make(pg, POLY, seed=9)
    ring = torch.full((6,), float("nan")).pin_memory()
    for t, (i, c) in enumerate(batches):
        a.train_step(torch.from_numpy(i).pin_memory(), torch.from_numpy(c).pin_memory(), 0.1, loss_out=ring[t:t + 1])
    a.sync()
    lb = [b.train_step(i, c, 0.1) for i, c in batches]
    assert np.array_equal(ring.numpy(), np.array(lb, np.float32))
    for x, y in zip(a.get_params()[:4], b.get_params()[:4]):
        assert np.array_equal(x, y)
    a.close(); b.close()


def test_cuda_graph_capture_replay_equals_eager(pg):
    """PG_OPT_RESERVE pre-sizes the workspace so steps with device inputs and a
    device loss can be captured in a CUDA graph; replaying the graph must give
    the same (DET: bitwise) parameters and losses as eager calls."""
    import torch
    V, d, n, h = POLY["V"], POLY["d"], POLY["n"], POLY["h"]
    B, K = 2048, 3
    bs = [synth.batch(V, n, B, seed=21, step=t) for t in range(K)]
    di = [torch.from_numpy(i).cuda() for i, _ in bs]
    dc = [torch.from_numpy(c).cuda() for _, c in bs]
    s = torch.cuda.Stream()
    eager = pg.PolyglotModel(V, d, n, h, seed=5, stream=s)
    graphed = pg.PolyglotModel(V, d, n, h, seed=5, stream=s)
    graphed.reserve(B)
    le = torch.zeros(K, device="cuda")
    lg = torch.zeros(K, device="cuda")
    with torch.cuda.stream(s):
        for t in range(K):
            eager.train_step(di[t], dc[t], 0.1, loss_out=le[t:t + 1])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(K):
            graphed.train_step(di[t], dc[t], 0.1, loss_out=lg[t:t + 1])
    # capture records the launches without running them: the parameters are
    # still the initial ones until the replay
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(le, lg)
    for a, b in zip(eager.get_params(), graphed.get_params()):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    eager.close(); graphed.close()


@pytest.mark.parametrize("scatter", [0, 1])
@pytest.mark.parametrize("fused", [True, False])
def test_nonfinite_loss_diverged_no_mutation(pg, scatter, fused):
    # a non-finite loss -> PG_EDIVERGED and no parameter changes.
    # Saturated units and w2 = 1e37: margins ~1e38, the fp32 hinge sum overflows.
    m = make(pg, POLY, seed=2, scatter=scatter, fused=fused)
    C, W1, b1, w2, b2 = m.get_params()
    big = (C, W1 * np.float32(1000), b1, np.full_like(w2, 1e37))
    m.set_params(*big, b2=b2)
    idx, corr = synth.batch(POLY["V"], POLY["n"], 512, seed=1)
    with pytest.raises(pg.PGError) as e:
        m.train_step(idx, corr, 0.1)
    assert e.value.status == pg.PG_EDIVERGED
    for a, b in zip(big, m.get_params()[:4]):
        assert np.array_equal(a, b)
    # the literal north-star form returns NaN
    assert np.isnan(pg.pg_train_step_loss(m.handle, idx, corr, 0.1))
    # asynchronous steps make it sticky until pg_sync
    m.train_step(idx, corr, 0.1, loss_out=None)
    with pytest.raises(pg.PGError) as e:
        m.sync()
    assert e.value.status == pg.PG_EDIVERGED
    m.sync()   # cleared
    m.set_params(C, W1, b1, w2, b2)
    m.train_step(idx, corr, 0.1)   # and the model keeps working
    m.close()


_PDL_SCRIPT = r"""
import sys, hashlib
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1404_1521_b200 as pg, synth
m = pg.PolyglotModel(100_000, 64, 5, 32, seed=3)
bs = [synth.batch(100_000, 5, 2048, seed=31, step=t) for t in range(8)]
di = [torch.from_numpy(i).cuda() for i, _ in bs]
dc = [torch.from_numpy(c).cuda() for _, c in bs]
loss = torch.zeros(8, device="cuda")
for t in range(8):
    m.train_step(di[t], dc[t], 0.5, loss_out=loss[t:t + 1])   # back to back, no host sync
m.sync()
h = hashlib.sha256(loss.cpu().numpy().tobytes())
for x in m.get_params()[:4]:
    h.update(np.ascontiguousarray(x).tobytes())
print(h.hexdigest())
"""


@pytest.mark.parametrize("pdl", ["0", "1"])
def test_pdl_launch_matches_cooperative_bitwise(pg, pdl):
    # PG_PDL=1 launches the step without the cooperative attribute, with
    # programmatic stream serialisation (step.cu launch_step_phases): eight
    # back-to-back DET steps must give the bits of the default launch
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("0", pdl):
        env = dict(os.environ, PG_PDL=v)
        r = subprocess.run([sys.executable, "-c", _PDL_SCRIPT, root], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out[pdl]
