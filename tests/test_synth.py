"""Input recipe checks."""
import numpy as np

import synth


def test_zipf_head_mass_matches_harmonic():
    V = 100_000
    ids = synth.zipf_ids(V, 1_000_000, 42, synth.S_SCATTER_I, 0)
    H = (1.0 / np.arange(1, V + 1)).sum()
    assert abs(H - 12.090) < 1e-3
    frac0 = (ids == 0).mean()
    assert abs(frac0 - 1 / H) < 0.002            # 8.27%
    assert ids.min() >= 0 and ids.max() < V


def test_batches_deterministic_and_valid():
    V, n, B = 1000, 5, 64
    a = synth.batch(V, n, B, seed=42, step=3)
    b = synth.batch(V, n, B, seed=42, step=3)
    c = synth.batch(V, n, B, seed=42, step=4)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert not (a[0] == c[0]).all()
    idx, corr = a
    assert idx.dtype == np.int32 and idx.shape == (B, n)
    assert (corr != idx[:, n // 2]).all()
    assert (idx[1:, :-1] == idx[:-1, 1:]).all()           # sliding windows (G14)


def test_scatter_int_payload_range():
    I, Y = synth.scatter_inputs(1000, 8, 5000, "uniform", "int")
    assert Y.min() == -8 and Y.max() == 8 and (Y == np.round(Y)).all()
    assert I.min() >= 0 and I.max() < 1000
