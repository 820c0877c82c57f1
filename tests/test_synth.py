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


def test_bigram_corpus_structure():
    """Convergence-study corpus: every transition is
    one of the word's `branching` successors; windows are contiguous corpus
    slices inside [lo, hi); corrupt centres differ from the centre."""
    V, br = 300, 4
    toks = synth.bigram_corpus(V, 20_000, seed=3, branching=br)
    assert toks.dtype == np.int32 and toks.min() >= 0 and toks.max() < V
    succ = {}
    for a, b in zip(toks[:-1], toks[1:]):
        succ.setdefault(int(a), set()).add(int(b))
    assert max(len(s) for s in succ.values()) <= br
    assert np.mean([len(s) for s in succ.values()]) > br - 1.5   # most words show several successors
    idx, corr = synth.corpus_batch(toks, V, 5, 500, seed=3, step=0, lo=1000, hi=5000)
    assert idx.shape == (500, 5) and (corr != idx[:, 2]).all()
    for w in idx[:50]:
        starts = np.flatnonzero(toks[1000:5000 - 4] == w[0]) + 1000
        assert any((toks[s:s + 5] == w).all() for s in starts)
