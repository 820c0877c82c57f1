"""Helpers for GPU-vs-oracle parity tests (test infrastructure).

Both sides receive the same seeded inputs from synth/ and the same float32
starting parameters; the oracle widens them to float64.  Tolerances follow
SURVEY.md §8(c) T1-T5.
"""
import numpy as np

import oracle
import synth


def oracle_from_gpu_params(params, V, d, n, h):
    C, W1, b1, w2, b2 = params
    return oracle.Params(V, d, n, h, C.astype(np.float64), W1.astype(np.float64),
                         b1.astype(np.float64), w2.astype(np.float64), float(b2))


def rel_inf(a, b):
    """||a - b||_inf / ||b||_inf (0 if both zero)."""
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    den = np.abs(b).max() if b.size else 0.0
    num = np.abs(a - b).max() if b.size else 0.0
    return 0.0 if den == 0.0 and num == 0.0 else num / max(den, 1e-300)


def num_sms():
    import torch
    return torch.cuda.get_device_properties(0).multi_processor_count


def chunk_row_counts(idx, corr, V, P, T):
    """Per embedding row: the number of (CTA, chunk) lists of one step that
    contain it -- exactly the number of red.global.add the ATOMIC step issues
    for the row (each chunk pre-sums its duplicates; CTA p owns examples
    [p*B/P, (p+1)*B/P) in chunks of T)."""
    B = corr.shape[0]
    cnt = np.zeros(V, np.int64)
    for p in range(P):
        lo, hi = p * B // P, (p + 1) * B // P
        for e0 in range(lo, hi, T):
            e1 = min(hi, e0 + T)
            cnt[np.unique(np.concatenate([idx[e0:e1].ravel(), corr[e0:e1]]))] += 1
    return cnt


def run_both(model, V, d, n, h, B, steps, lr=0.1, seed=42, kind="sliding", start_params=None,
             step0=0, chunk_T=32):
    """Drive the GPU model and the oracle through the same `steps` SGD steps.

    Returns (gpu_losses, ref_losses, p0 (float32 tuple), gpu_params_end, oracle Params).
    run_both.roundings: per embedding row, the red.adds an ATOMIC step issues
    (chunk_row_counts summed over the steps; chunk_T = the path's chunk size)."""
    import paper_1404_1521_b200 as pg
    if start_params is not None:
        pg.pg_set_params(model.handle, *start_params[:4], b2=start_params[4])
    p0 = pg.pg_get_params(model.handle)
    ref = oracle_from_gpu_params(p0, V, d, n, h)
    gl, rl = [], []
    rnd = np.zeros(V, np.int64)     # red.adds per embedding row (ATOMIC roundings)
    P = min(num_sms(), B)
    for t in range(steps):
        idx, corr = synth.batch(V, n, B, seed=seed, step=step0 + t, kind=kind)
        gl.append(model.train_step(idx, corr, lr))
        rl.append(oracle.train_step(ref, idx, corr, lr))
        rnd += chunk_row_counts(idx, corr, V, P, chunk_T)
    run_both.roundings = rnd
    return np.array(gl), np.array(rl), p0, pg.pg_get_params(model.handle), ref


def assert_parity(gl, rl, p0, pend, ref, tau_delta=1e-3, tol=1e-4, c_roundings=None):
    """T1 per-step loss, T2 per-tensor state, T3 per-tensor deltas, T4 b2.

    T3 allows, per element, the float32 STORAGE rounding of the GPU state:
    each step stores theta in float32 (north_star mandates fp32 parameters),
    which costs at most half an ulp of the stored value per step.  At default
    init an embedding update is ~0.1 ulp of |C| ~ 0.5, so without this
    allowance the delta check measures storage rounding, not the kernel
    (DESIGN.md "Parity tolerances").  The saturated-regime test keeps updates
    far above the storage floor and runs with tau = 1e-4.  In atomic mode every
    red.add rounds the stored row, so c_roundings (per embedding row: the
    number of red.adds issued, run_both.roundings) replaces `steps`."""
    rel_loss = np.abs(gl - rl) / np.maximum(np.abs(rl), 1e-30)
    assert rel_loss.max() <= tol, f"T1 loss rel err {rel_loss.max():.3g}"
    C, W1, b1, w2, b2 = pend
    pairs = {"C": (C, ref.C, p0[0]), "W1": (W1, ref.W1, p0[1]), "b1": (b1, ref.b1, p0[2]),
             "w2": (w2, ref.w2, p0[3])}
    report = {}
    for k, (g, r, z) in pairs.items():
        e_state = rel_inf(g, r)
        dg = g.astype(np.float64) - z.astype(np.float64)
        dr = r - z.astype(np.float64)
        steps = len(gl)
        ulp = np.maximum(np.spacing(np.abs(z).astype(np.float32)),
                         np.spacing(np.abs(g).astype(np.float32))).astype(np.float64)
        nround = steps
        if k == "C" and c_roundings is not None:
            nround = np.maximum(c_roundings, steps)[:, None]
        excess = np.maximum(np.abs(dg - dr) - 0.5 * nround * ulp, 0.0)
        e_delta = excess.max() / max(np.abs(dr).max(), 1e-300)
        report[k] = (e_state, e_delta)
        assert e_state <= tol, f"T2 {k}: {e_state:.3g}"
        if np.abs(dr).max() > 0:
            assert e_delta <= tau_delta, f"T3 {k} delta: {e_delta:.3g}"
    assert b2 == p0[4], "T4: b2 must never change"
    return report


def higham_bound(W0, Y, I):
    """Rigorous bound on |fp32 W[I] += Y - exact| per element, for ANY
    summation order of a row's m contributions (W0 included): gamma_m *
    (|W0| + sum |Y|) with gamma_m = m u / (1 - m u), u = 2^-24 (Higham,
    recursive summation), plus the fp32 rounding of the stored result."""
    u = 2.0 ** -24
    I = np.asarray(I, np.int64)
    absum = np.abs(W0).astype(np.float64)
    np.add.at(absum, I, np.abs(Y).astype(np.float64))
    m = np.ones(W0.shape[0], np.float64)
    np.add.at(m, I, 1.0)
    gam = (m * u / (1 - m * u))[:, None]
    return gam * absum + u * absum
