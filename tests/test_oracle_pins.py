"""Pins for the float64 CPU oracle (oracle/pgo.c) against things other than itself.

Each test names what fixes the expected value: a worked example printed in
SPEC.md (tests/golden/spec_examples.json), published SplitMix64 vectors, a
closed form, an invariant, central finite differences, or an independently
written dense one-hot evaluator (no index arithmetic in its algebra).
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- scatter-add
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_index_add_spec_examples(dtype):
    for ex in _gold("spec_examples.json")["index_add"]:
        W = np.array(ex["W"], dtype=dtype)
        cols = W.shape[1]
        Y = np.array(ex["Y"], dtype=dtype).reshape(-1, cols)
        oracle.index_add(W, Y, np.array(ex["I"], dtype=np.int32))
        np.testing.assert_array_equal(W, np.array(ex["expect"], dtype=dtype), err_msg=ex["cite"])


def test_index_add_10000_ones_exact():
    g = _gold("spec_examples.json")["ones_10000"]
    W = np.zeros((g["rows"], g["cols"]), dtype=np.float32)
    oracle.index_add(W, np.ones((g["n"], g["cols"]), np.float32), np.zeros(g["n"], np.int32))
    assert (W == g["expect"]).all()


def test_index_add_out_of_range_leaves_w_unchanged():
    W = np.arange(6, dtype=np.float64).reshape(3, 2)
    W0 = W.copy()
    with pytest.raises(oracle.OracleError) as e:
        oracle.index_add(W, np.ones((3, 2)), np.array([0, 3, 1], np.int32))
    assert e.value.status == 2 and "position 1, value 3" in str(e.value)
    np.testing.assert_array_equal(W, W0)


def test_index_add_decomposable_and_local():
    # index_add(y1++y2, i1++i2) == index_add(y1,i1); index_add(y2,i2);
    # rows outside I bit-identical.
    rng = np.random.default_rng(0)
    W = rng.standard_normal((20, 3))
    I = rng.integers(0, 10, 15).astype(np.int32)
    Y = rng.standard_normal((15, 3))
    A = oracle.index_add(W.copy(), Y, I)
    Bm = oracle.index_add(oracle.index_add(W.copy(), Y[:7], I[:7]), Y[7:], I[7:])
    np.testing.assert_array_equal(A, Bm)
    np.testing.assert_array_equal(A[10:], W[10:])
    # agrees with numpy's unbuffered add.at (a library routine, same k order)
    C = W.copy(); np.add.at(C, I, Y)
    np.testing.assert_array_equal(A, C)


# ---------------------------------------------------------------- init spec
def test_splitmix64_published_vectors():
    g = _gold("splitmix64_vectors.json")
    got = synth.splitmix64_raw(g["seed"], 5)
    assert [int(v) for v in got] == [int(s) for s in g["outputs"]]


def test_init_follows_spec():
    # reading G10: value = float32((2u-1) r), u = (x>>40)/2^24, stream keyed by
    # seed ^ (0x632BE59BD9B4E019 * (tensor_id+1)); recomputed here with the
    # independently written numpy SplitMix64 pinned above.
    V, d, n, h, seed = 37, 4, 5, 6, 1234
    p = oracle.Params.init(V, d, n, h, seed)
    for tid, arr, r in ((0, p.C, 0.5), (1, p.W1, 0.5 / (n * d)), (2, p.w2, 0.5 / h)):
        key = seed ^ ((0x632BE59BD9B4E019 * (tid + 1)) & 0xFFFFFFFFFFFFFFFF)
        x = synth.splitmix64_raw(key, arr.size)
        u = (x >> np.uint64(40)).astype(np.float64) / 16777216.0
        exp = ((2.0 * u - 1.0) * r).astype(np.float32).astype(np.float64)
        np.testing.assert_array_equal(arr.ravel(), exp)
    assert (p.b1 == 0).all() and p.b2[0] == 0.0


def test_init_ranges_and_moments():
    V, d, n, h = 4000, 16, 5, 32
    p = oracle.Params.init(V, d, n, h, 42)
    assert np.abs(p.C).max() <= 0.5 and np.abs(p.W1).max() <= 0.5 / (n * d)
    assert np.abs(p.w2).max() <= 0.5 / h
    # U[-r, r): mean 0, variance r^2/3
    assert abs(p.C.mean()) < 0.01 and abs(p.C.var() - 0.25 / 3) < 0.002


# ---------------------------------------------------------------- closed forms
def test_zero_params_loss_one_and_fixed_point():
    V, d, n, h = 30, 4, 5, 8
    p = oracle.Params(V, d, n, h)
    idx, corr = synth.batch(V, n, 16, seed=3)
    assert oracle.loss(p, idx, corr) == 1.0
    for _ in range(3):
        assert oracle.train_step(p, idx, corr, 0.1) == 1.0
    assert not p.flat().any()                        # SPEC.md:228,237 zero grads


def test_score_clamp_case():
    # SPEC.md:211 in hardtanh form: h=1, W1=0, b1=[c], w2=[1], b2=0 -> clamp(c)
    V, d, n = 7, 3, 5
    idx, _ = synth.batch(V, n, 4, seed=5, kind="uniform")
    for c in _gold("spec_examples.json")["score"][1]["c"]:
        p = oracle.Params(V, d, n, 1, C=np.ones((V, d)), b1=[c], w2=[1.0])
        assert (oracle.score(p, idx) == min(1.0, max(-1.0, c))).all()
    p = oracle.Params(V, d, n, 3)
    assert (oracle.score(p, idx) == 0.0).all()


def _centre_model(C_col, W1_centre, w2, n=3, b1=None):
    """d=1 model whose hidden pre-activation is W1_centre * C[centre]."""
    V = len(C_col)
    h = len(W1_centre)
    W1 = np.zeros((n, h)); W1[n // 2] = W1_centre
    return oracle.Params(V, 1, n, h, C=np.array(C_col, float).reshape(V, 1), W1=W1,
                         b1=b1, w2=w2)


def test_hinge_inactive_zero_loss_no_change():
    # s >= s' + 1 everywhere -> loss 0, params unchanged
    p = _centre_model([0.9, -0.9, 0.0], [1.0], [1.0])
    idx = np.array([[2, 0, 2], [0, 0, 1]], np.int32)
    corr = np.array([1, 1], np.int32)
    q = p.copy()
    assert oracle.train_step(q, idx, corr, 0.5) == 0.0
    np.testing.assert_array_equal(q.flat(), p.flat())


def test_hinge_kink_zero_subgradient():
    # reading G3: m = 0 exactly -> inactive.  s - s' = 0.5 - (-0.5) = 1.
    p = _centre_model([0.5, -0.5, 0.25], [1.0], [1.0])
    idx = np.array([[2, 0, 2]], np.int32)
    corr = np.array([1], np.int32)
    f = oracle.forward(p, idx, corr)
    assert 1.0 - f["s"][0] + f["s_corr"][0] == 0.0 and f["loss"] == 0.0
    g = oracle.backward(p, idx, corr)
    assert len(g["rows"]) == 0 and not g["dW1"].any() and not g["dw2"].any()


def test_hardtanh_kink_zero_derivative():
    # reading G2: |a| = 1 exactly -> hardtanh' = 0.  Unit 0: a = 1 (true), a' = 0.25.
    p = _centre_model([1.0, 0.25, 0.0], [1.0], [0.5])
    idx = np.array([[2, 0, 2]], np.int32)
    corr = np.array([1], np.int32)
    f = oracle.forward(p, idx, corr)
    assert f["a"][0, 0] == 1.0 and f["a_corr"][0, 0] == 0.25
    g = oracle.backward(p, idx, corr)
    # only the corrupt window passes gradient: dW1[centre] = x'_c * (+1/B) * w2
    assert g["dW1"][1, 0] == 0.25 * 0.5
    assert g["db1"][0] == 0.5
    # true-window rows carry zero gradient, corrupt centre row carries W1_c delta'
    assert (g["Y"][:3] == 0).all() and g["Y"][4, 0] == 0.5 and g["rows"][4] == 1


def test_saturated_only_w2_moves_exactly():
    # all |a|,|a'| > 1 -> delta = delta' = 0; w2 -= lr * sum_k (-1/B)(z_k - z'_k);
    # exact in fp64 for dyadic lr/B.
    C = [2.0, -2.0, 3.0, -3.0]
    p = _centre_model(C, [1.0, -1.0], [0.5, 0.25])
    idx = np.array([[0, 0, 0], [1, 1, 1], [2, 3, 2], [3, 2, 1]], np.int32)
    corr = np.array([1, 2, 3, 0], np.int32)
    q = p.copy()
    lr, B = 0.5, 4
    loss = oracle.train_step(q, idx, corr, lr)
    zc = np.sign(np.array(C))[idx[:, 1]]
    zcc = np.sign(np.array(C))[corr]
    z = np.stack([zc, -zc], 1); zp = np.stack([zcc, -zcc], 1)
    s = z @ p.w2; sp = zp @ p.w2
    assert loss == np.mean(np.maximum(0, 1 - s + sp))
    exp_w2 = p.w2 - lr * ((-1.0 / B) * (z - zp)).sum(0)
    np.testing.assert_array_equal(q.w2, exp_w2)
    np.testing.assert_array_equal(q.C, p.C)
    np.testing.assert_array_equal(q.W1, p.W1)
    np.testing.assert_array_equal(q.b1, p.b1)


def test_swap_symmetry():
    # swapping positive and negative maps m -> 2 - m
    V, d, n, h = 40, 5, 5, 7
    C, W1, b1, w2, b2 = synth.random_params(V, d, n, h, seed=9, w1_scale=0.3, w2_scale=1.0)
    p = oracle.Params(V, d, n, h, C, W1, b1, w2, b2)
    idx, corr = synth.batch(V, n, 32, seed=4, kind="uniform")
    f = oracle.forward(p, idx, corr)
    idx2 = idx.copy(); idx2[:, n // 2] = corr
    f2 = oracle.forward(p, idx2, idx[:, n // 2])
    m = 1 - f["s"] + f["s_corr"]; m2 = 1 - f2["s"] + f2["s_corr"]
    np.testing.assert_allclose(m2, 2 - m, rtol=0, atol=1e-14)


def test_b2_invariant_and_locality():
    V, d, n, h = 500, 8, 5, 16
    p = oracle.Params.init(V, d, n, h, 7)
    p.b2[0] = 0.375
    idx, corr = synth.batch(V, n, 32, seed=11)
    q = p.copy()
    oracle.train_step(q, idx, corr, 0.1)
    assert q.b2[0] == 0.375                          # db2 = g + g' = 0 term by term
    touched = np.zeros(V, bool); touched[idx.ravel()] = True; touched[corr] = True
    np.testing.assert_array_equal(q.C[~touched], p.C[~touched])
    assert (q.C[touched] != p.C[touched]).any()


def test_errors_no_mutation():
    V, d, n, h = 20, 4, 5, 8
    p = oracle.Params.init(V, d, n, h, 1)
    idx, corr = synth.batch(V, n, 8, seed=2)
    bad = idx.copy(); bad[3, 1] = V
    q = p.copy()
    with pytest.raises(oracle.OracleError) as e:
        oracle.train_step(q, bad, corr, 0.1)
    assert e.value.status == 2 and f"position {3 * n + 1}, value {V}" in str(e.value)
    badc = corr.copy(); badc[5] = -1
    with pytest.raises(oracle.OracleError) as e:
        oracle.train_step(q, idx, badc, 0.1)
    assert e.value.status == 2 and f"position {8 * n + 5}" in str(e.value)
    np.testing.assert_array_equal(q.flat(), p.flat())
    with pytest.raises(oracle.OracleError) as e:
        oracle.train_step(q, idx, corr, -0.1)
    assert e.value.status == 1


# ---------------------------------------------------------------- dense one-hot evaluator
def dense_onehot(p, idx, corr):
    """Independent evaluator: windows as one-hot selection matrices S (B, n, V),
    x = S C, gradients by matrix algebra, dC = sum_p S_p^T dX_p."""
    B, n = idx.shape
    V, d = p.C.shape
    c = n // 2
    S = (idx[:, :, None] == np.arange(V)[None, None, :]).astype(float)
    Sc = S.copy()
    Sc[:, c, :] = (corr[:, None] == np.arange(V)[None, :])
    X = np.einsum("bpv,vd->bpd", S, p.C).reshape(B, n * d)
    Xc = np.einsum("bpv,vd->bpd", Sc, p.C).reshape(B, n * d)
    A = X @ p.W1 + p.b1
    Ac = Xc @ p.W1 + p.b1
    Z, Zc = np.clip(A, -1, 1), np.clip(Ac, -1, 1)
    s, sc = Z @ p.w2 + p.b2[0], Zc @ p.w2 + p.b2[0]
    m = 1 - s + sc
    L = np.maximum(m, 0).mean()
    act = (m > 0).astype(float)
    g, gc = -act / B, act / B
    D = g[:, None] * p.w2[None, :] * (np.abs(A) < 1)
    Dc = gc[:, None] * p.w2[None, :] * (np.abs(Ac) < 1)
    dW1 = X.T @ D + Xc.T @ Dc
    db1 = (D + Dc).sum(0)
    dw2 = Z.T @ g + Zc.T @ gc
    dX = (D @ p.W1.T).reshape(B, n, d)
    dXc = (Dc @ p.W1.T).reshape(B, n, d)
    dC = np.einsum("bpv,bpd->vd", S, dX) + np.einsum("bpv,bpd->vd", Sc, dXc)
    return L, dict(C=dC, W1=dW1, b1=db1, w2=dw2, b2=(g + gc).sum()), A, Ac, m


def oracle_dense_grads(p, idx, corr):
    g = oracle.backward(p, idx, corr)
    dC = np.zeros_like(p.C)
    np.add.at(dC, g["rows"], g["Y"])
    return dict(C=dC, W1=g["dW1"], b1=g["db1"], w2=g["dw2"], b2=g["db2"])


def _saturating_fixture(seed, V=50, d=8, n=5, h=16, B=6, w1x=60.0, w2x=40.0):
    C, W1, b1, w2, b2 = synth.random_params(V, d, n, h, seed, w1_scale=w1x * 0.5 / (n * d),
                                            w2_scale=w2x * 0.5 / h, b1_scale=0.3, b2=0.1)
    p = oracle.Params(V, d, n, h, C, W1, b1, w2, b2)
    idx, corr = synth.batch(V, n, B, seed=seed + 1000, kind="uniform")
    return p, idx, corr


def test_brute_force_tiny_vocab_all_windows():
    # SURVEY.md §8(c) pin (ii): V=5, d=2, n=3, h=2; every one of the
    # V^n windows x every corrupt centre != true centre, as one full batch.
    V, d, n, h = 5, 2, 3, 2
    C, W1, b1, w2, b2 = synth.random_params(V, d, n, h, 77, w1_scale=1.5, w2_scale=1.0,
                                            b1_scale=0.5, b2=0.2)
    p = oracle.Params(V, d, n, h, C, W1, b1, w2, b2)
    wins = np.array(np.meshgrid(*[np.arange(V)] * n, indexing="ij")).reshape(n, -1).T
    idx, corr = [], []
    for w in wins:
        for cw in range(V):
            if cw != w[n // 2]:
                idx.append(w); corr.append(cw)
    idx = np.array(idx, np.int32); corr = np.array(corr, np.int32)
    assert idx.shape[0] == V ** n * (V - 1)
    L, G, A, Ac, m = dense_onehot(p, idx, corr)
    assert abs(oracle.loss(p, idx, corr) - L) <= 1e-14 * max(1, abs(L))
    f = oracle.forward(p, idx, corr)
    np.testing.assert_allclose(f["a"], A, rtol=0, atol=1e-14)
    np.testing.assert_allclose(f["a_corr"], Ac, rtol=0, atol=1e-14)
    O = oracle_dense_grads(p, idx, corr)
    for k in G:
        np.testing.assert_allclose(O[k], G[k], rtol=1e-12, atol=1e-15, err_msg=k)


def _fd_check(p, idx, corr, rel=1e-5, absf=1e-8):
    an = oracle_dense_grads(p, idx, corr)
    flat_an = np.concatenate([an["C"].ravel(), an["W1"].ravel(), an["b1"], an["w2"], [an["b2"]]])
    fields = [("C", p.C), ("W1", p.W1), ("b1", p.b1), ("w2", p.w2), ("b2", p.b2)]
    fd = []
    for _, arr in fields:
        flat = arr.reshape(-1)
        for i in range(flat.size):
            t = flat[i]
            hstep = 1e-6 * max(1.0, abs(t))
            flat[i] = t + hstep; lp = oracle.loss(p, idx, corr)
            flat[i] = t - hstep; lm = oracle.loss(p, idx, corr)
            flat[i] = t
            fd.append((lp - lm) / (2 * hstep))
    fd = np.array(fd)
    err = np.abs(fd - flat_an)
    tol = rel * np.maximum(np.abs(fd), np.abs(flat_an)) + absf
    assert (err <= tol).all(), f"max excess {np.max(err - tol)} at {np.argmax(err - tol)}"
    return flat_an


def test_finite_differences_20_random_models():
    # central FD in fp64, step 1e-6 max(1,|theta|),
    # 1e-5 relative with a 1e-8 absolute floor.  W1/w2 scaled so that some
    # units saturate and some margins go negative; fixtures near a kink rejected.
    good, seed = 0, 100
    saw_sat = saw_inactive = False
    while good < 20:
        seed += 1
        p, idx, corr = _saturating_fixture(seed)
        f = oracle.forward(p, idx, corr)
        m = 1 - f["s"] + f["s_corr"]
        kinks = min(np.abs(m).min(), np.abs(np.abs(f["a"]) - 1).min(),
                    np.abs(np.abs(f["a_corr"]) - 1).min())
        if kinks < 1e-4:
            continue
        saw_sat |= bool((np.abs(f["a"]) > 1).any())
        saw_inactive |= bool((m < 0).any())
        g = _fd_check(p, idx, corr)
        assert np.abs(g).max() > 0
        good += 1
    assert saw_sat and saw_inactive


def test_dp_emulation_equals_single_step():
    V, d, n, h = 300, 8, 5, 16
    p = oracle.Params.init(V, d, n, h, 5)
    idx, corr = synth.batch(V, n, 64, seed=8)
    a, b = p.copy(), p.copy()
    la = oracle.train_step(a, idx, corr, 0.1)
    lb = oracle.train_step_dp(b, idx, corr, 0.1, world=4)
    assert abs(la - lb) <= 1e-14
    np.testing.assert_allclose(b.flat(), a.flat(), rtol=1e-13, atol=1e-16)


# ---------------------------------------------------------------- tanh variant
def test_tanh_score_closed_form():
    # SPEC.md:211 with the spec's own nonlinearity: h=1, W1=0,
    # b1=[c], w2=[1], b2=0 -> s = tanh(c) for every window
    V, d, n = 7, 3, 5
    idx, _ = synth.batch(V, n, 4, seed=5, kind="uniform")
    with oracle.activation(oracle.TANH):
        for c in (-3.0, -1.0, -0.25, 0.0, 0.5, 1.0, 2.0):
            p = oracle.Params(V, d, n, 1, C=np.ones((V, d)), b1=[c], w2=[1.0])
            np.testing.assert_allclose(oracle.score(p, idx), np.tanh(c), rtol=0, atol=1e-15)
    p = oracle.Params(V, d, n, 1, C=np.ones((V, d)), b1=[3.0], w2=[1.0])
    assert (oracle.score(p, idx) == 1.0).all()      # the switch is restored (hardtanh clamps)


def test_tanh_zero_params_fixed_point():
    V, d, n, h = 30, 4, 5, 8
    p = oracle.Params(V, d, n, h)
    idx, corr = synth.batch(V, n, 16, seed=3)
    with oracle.activation(oracle.TANH):
        for _ in range(2):
            assert oracle.train_step(p, idx, corr, 0.1) == 1.0
    assert not p.flat().any()


def test_tanh_finite_differences():
    # tanh is smooth: only the hinge kink m = 0 has to be avoided.  Large
    # weights make some units saturate (tanh' ~ 0) and some margins negative.
    good, seed = 0, 500
    saw_sat = saw_inactive = False
    with oracle.activation(oracle.TANH):
        while good < 8:
            seed += 1
            p, idx, corr = _saturating_fixture(seed, w1x=120.0)
            f = oracle.forward(p, idx, corr)
            m = 1 - f["s"] + f["s_corr"]
            if np.abs(m).min() < 1e-4:
                continue
            saw_sat |= bool((np.abs(f["a"]) > 2).any())
            saw_inactive |= bool((m < 0).any())
            g = _fd_check(p, idx, corr)
            assert np.abs(g).max() > 0
            good += 1
    assert saw_sat and saw_inactive


def test_tanh_differs_from_hardtanh_inside():
    # the switch really changes the arithmetic (|a| < 1: tanh(a) != a)
    V, d, n, h = 40, 4, 5, 6
    p = oracle.Params.init(V, d, n, h, 3)
    p.W1 *= 30
    idx, corr = synth.batch(V, n, 8, seed=4)
    l_hard = oracle.loss(p, idx, corr)
    with oracle.activation(oracle.TANH):
        l_tanh = oracle.loss(p, idx, corr)
    assert abs(l_hard - l_tanh) > 1e-6


# ---------------------------------------------------------------- sum reduction (reading G4 alternative)
def test_sum_reduction_identities():
    # sum_k l_k = B * mean, and (exact for B a power of two) one SGD step of the
    # summed loss at lr is the mean step at lr * B
    V, d, n, h, B = 60, 4, 5, 8, 16
    p = oracle.Params.init(V, d, n, h, 9)
    p.W1 *= 40
    idx, corr = synth.batch(V, n, B, seed=2)
    a, b = p.copy(), p.copy()
    lm = oracle.train_step(a, idx, corr, 0.25 * B)
    with oracle.reduction(oracle.SUM):
        ls = oracle.train_step(b, idx, corr, 0.25)
    assert ls == lm * B
    np.testing.assert_array_equal(a.flat(), b.flat())
    assert oracle.loss(p, idx, corr) == lm         # switch restored


def test_sum_reduction_finite_differences():
    with oracle.reduction(oracle.SUM):
        for seed in (601, 602, 603):
            p, idx, corr = _saturating_fixture(seed)
            f = oracle.forward(p, idx, corr)
            m = 1 - f["s"] + f["s_corr"]
            if min(np.abs(m).min(), np.abs(np.abs(f["a"]) - 1).min(), np.abs(np.abs(f["a_corr"]) - 1).min()) < 1e-4:
                continue
            _fd_check(p, idx, corr)


def test_sum_reduction_dp_emulation():
    V, d, n, h = 300, 8, 5, 16
    p = oracle.Params.init(V, d, n, h, 5)
    idx, corr = synth.batch(V, n, 64, seed=8)
    a, b = p.copy(), p.copy()
    with oracle.reduction(oracle.SUM):
        la = oracle.train_step(a, idx, corr, 0.01)
        lb = oracle.train_step_dp(b, idx, corr, 0.01, world=4)
    assert abs(la - lb) <= 1e-12 * abs(la)
    np.testing.assert_allclose(b.flat(), a.flat(), rtol=1e-13, atol=1e-16)


# ---------------------------------------------------------------- update rule
def test_sgd_update_spec_examples():
    ex0, ex1 = _gold("spec_examples.json")["sgd_update"]
    # zero gradients -> every parameter unchanged
    V, d, n, h = 9, 3, 5, 4
    p = oracle.Params.init(V, d, n, h, 3)
    p.b2[0] = 0.25
    q = p.copy()
    oracle.sgd_update(q, {"rows": np.array(ex0["rows"], np.int32), "Y": np.zeros((0, d))}, ex0["lr"])
    np.testing.assert_array_equal(q.flat(), p.flat(), err_msg=ex0["cite"])
    # lr = 1, one sparse row -> that embedding row decreased by exactly the row
    C = np.array(ex1["C"])
    p = oracle.Params(C.shape[0], C.shape[1], 1, 1, C=C)
    oracle.sgd_update(p, {"rows": np.array(ex1["rows"], np.int32), "Y": np.array(ex1["Y"])}, ex1["lr"])
    np.testing.assert_array_equal(p.C, np.array(ex1["expect_C"]), err_msg=ex1["cite"])


def test_sgd_update_dense_direction_and_scale():
    # SPEC.md:234 "theta -= lr * grad": with lr = 0.5 and gradients 2 * e_i the
    # parameter moves by exactly -1 (dyadic, exact in fp64) -- a sign or scale
    # error in any dense tensor moves it the wrong way.
    V, d, n, h = 4, 2, 3, 2
    p = oracle.Params(V, d, n, h)
    g = {"dW1": np.zeros((n * d, h)), "db1": np.zeros(h), "dw2": np.zeros(h), "db2": 0.0}
    g["dW1"][4, 1] = 2.0; g["db1"][0] = 2.0; g["dw2"][1] = 2.0
    oracle.sgd_update(p, g, 0.5)
    assert p.W1[4, 1] == -1.0 and p.b1[0] == -1.0 and p.w2[1] == -1.0
    assert np.count_nonzero(p.flat()) == 3
    # duplicated sparse rows accumulate: two rows of +1 at lr 0.25 -> -0.5
    oracle.sgd_update(p, {"rows": np.array([2, 2], np.int32), "Y": np.ones((2, d))}, 0.25)
    np.testing.assert_array_equal(p.C[2], [-0.5, -0.5])
    assert not p.C[[0, 1, 3]].any()


def test_sgd_update_bad_row_no_mutation():
    p = oracle.Params.init(6, 2, 3, 2, 1)
    q = p.copy()
    with pytest.raises(oracle.OracleError) as e:
        oracle.sgd_update(q, {"dW1": np.ones((6, 2)), "rows": np.array([1, 6], np.int32),
                              "Y": np.ones((2, 2))}, 0.1)
    assert e.value.status == 2
    np.testing.assert_array_equal(q.flat(), p.flat())


def _fd_grad(p, idx, corr):
    """Central finite differences of the loss for every parameter (no pgo_backward)."""
    out = []
    for arr in (p.C, p.W1, p.b1, p.w2):
        flat = arr.reshape(-1)
        g = np.empty(flat.size)
        for i in range(flat.size):
            t = flat[i]
            hs = 1e-6 * max(1.0, abs(t))
            flat[i] = t + hs; lp = oracle.loss(p, idx, corr)
            flat[i] = t - hs; lm = oracle.loss(p, idx, corr)
            flat[i] = t
            g[i] = (lp - lm) / (2 * hs)
        out.append(g.reshape(arr.shape))
    return out


def test_train_step_is_theta_minus_lr_fd_gradient():
    # One pgo_train_step must equal theta - lr * g for C, W1, b1, w2 with g the
    # central finite-difference gradient of the loss: a
    # sign, scale or index error in the update of any tensor (the embedding
    # update included) fails here independently of pgo_backward.
    good, seed = 0, 700
    while good < 5:
        seed += 1
        p, idx, corr = _saturating_fixture(seed)
        f = oracle.forward(p, idx, corr)
        m = 1 - f["s"] + f["s_corr"]
        if min(np.abs(m).min(), np.abs(np.abs(f["a"]) - 1).min(), np.abs(np.abs(f["a_corr"]) - 1).min()) < 1e-4:
            continue
        if not (m > 0).any():
            continue
        gfd = _fd_grad(p, idx, corr)
        lr = 0.375
        q = p.copy()
        oracle.train_step(q, idx, corr, lr)
        for name, g, before, after in zip(("C", "W1", "b1", "w2"), gfd, (p.C, p.W1, p.b1, p.w2),
                                          (q.C, q.W1, q.b1, q.w2)):
            assert np.abs(g).max() > 0, name
            step = after - before
            tol = 1e-5 * lr * np.maximum(np.abs(g), np.abs(g).max() * 1e-3) + 1e-9
            err = np.abs(step + lr * g)
            assert (err <= tol).all(), f"{name}: max err {err.max():.3g} (seed {seed})"
        assert q.b2[0] == p.b2[0]
        good += 1


def test_nonfinite_loss_is_diverged_and_changes_nothing():
    # a non-finite loss is a divergence error and no parameter
    # changes.  Saturated units and w2 = 3e307: margins reach ~1e308 and the
    # hinge sum overflows float64.
    V, d, n, h = 60, 4, 5, 8
    p = oracle.Params.init(V, d, n, h, 4)
    p.W1 *= 1000.0
    p.w2[:] = 3e307
    idx, corr = synth.batch(V, n, 64, seed=6)
    q = p.copy()
    with pytest.raises(oracle.OracleError) as e:
        oracle.train_step(q, idx, corr, 0.1)
    assert e.value.status == 6
    np.testing.assert_array_equal(q.flat(), p.flat())
    with pytest.raises(oracle.OracleError) as e:
        oracle.train_step_dp(q, idx, corr, 0.1, world=2)
    assert e.value.status == 6
    np.testing.assert_array_equal(q.flat(), p.flat())
