"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic: it only draws integers and
floats from a counter-based SplitMix64 stream and shapes them like the paper's
workload (SURVEY.md §8(d) "Synthetic inputs"):

  * token stream: Zipf(s=1) over ranks 1..V by inverse CDF, id = rank - 1
    (reading G13: frequency-sorted vocabulary);
  * windows: slide over B + n - 1 consecutive stream tokens per step (G14), or
    i.i.d. positions (stress variant);
  * corrupt centres: uniform on [0, V), rejection-resampled until != centre
    (SPEC.md:251);
  * scatter microbench: I ~ Zipf or uniform over the table rows, Y ~ U[-1, 1)
    float32 or integer-valued in [-8, 8] (the exact-sum mode);
  * random parameter sets for parity cases (the library's pg_set_params and
    the oracle receive the same float32 values);
  * a bigram-structured corpus for the convergence study (SURVEY.md §8(f)
    NEXT-1): a first-order Markov chain in which every word has `branching`
    successors, the next token uniform among them.

Every draw is a pure function of (seed, stream id, step, element index).
"""
from __future__ import annotations

import functools

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids (any distinct constants)
S_TOKENS, S_CORRUPT, S_IID, S_SCATTER_I, S_SCATTER_Y, S_PARAMS = 11, 12, 13, 21, 22, 31
S_BIGRAM_SUCC, S_BIGRAM_WALK, S_BIGRAM_POS = 41, 42, 43


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64_raw(state: int, count: int) -> np.ndarray:
    """The first `count` outputs of Vigna's SplitMix64 generator started at `state`."""
    i = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(np.uint64(state & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN)


def stream_key(seed: int, stream: int, step: int = 0) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        k = _mix(np.array([k ^ np.uint64((stream * 0x2545F4914F6CDD1D) & 0xFFFFFFFFFFFFFFFF)],
                          dtype=np.uint64) + GOLDEN)[0]
        k = _mix(np.array([k ^ np.uint64(step & 0xFFFFFFFFFFFFFFFF)], dtype=np.uint64) + GOLDEN)[0]
    return k


def bits(seed: int, stream: int, step: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of the SplitMix64 stream keyed by (seed, stream, step)."""
    key = stream_key(seed, stream, step)
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(key + i * GOLDEN)


def uniform01(seed, stream, step, count, start=0) -> np.ndarray:
    """float64 in [0, 1) with 53 random bits."""
    return (bits(seed, stream, step, start, count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@functools.lru_cache(maxsize=8)
def _zipf_cdf(V: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** s
    c = np.cumsum(w)
    return c / c[-1]


def zipf_ids(V: int, count: int, seed: int, stream: int, step: int, s: float = 1.0,
             start: int = 0) -> np.ndarray:
    """Zipf(s) ids in [0, V): P(id = r-1) proportional to r^-s (inverse CDF)."""
    u = uniform01(seed, stream, step, count, start)
    ids = np.searchsorted(_zipf_cdf(V, s), u, side="right")
    return np.minimum(ids, V - 1).astype(np.int32)


def uniform_ids(V: int, count: int, seed: int, stream: int, step: int, start: int = 0) -> np.ndarray:
    b = bits(seed, stream, step, start, count)
    return (b % np.uint64(V)).astype(np.int32)


def corrupt_centres(V: int, centres: np.ndarray, seed: int, step: int) -> np.ndarray:
    """Uniform on [0, V) and != centre, by rejection resampling."""
    B = centres.shape[0]
    out = uniform_ids(V, B, seed, S_CORRUPT, step)
    attempt = 1
    bad = out == centres
    while bad.any():
        redraw = uniform_ids(V, B, seed, S_CORRUPT, step, start=attempt * B)
        out = np.where(bad, redraw, out)
        bad = out == centres
        attempt += 1
    return out.astype(np.int32)


def batch(V: int, n: int, B: int, seed: int = 42, step: int = 0, kind: str = "sliding",
          zipf_s: float = 1.0):
    """(idx [B][n] int32, corr [B] int32) for SGD step `step`.

    kind="sliding": windows slide over a Zipf token stream of B+n-1 tokens
    (reading G14); kind="iid": every position drawn independently;
    kind="uniform": every position uniform (no Zipf skew)."""
    if kind == "sliding":
        toks = zipf_ids(V, B + n - 1, seed, S_TOKENS, step, zipf_s)
        idx = np.lib.stride_tricks.sliding_window_view(toks, n)[:B].copy()
    elif kind == "iid":
        idx = zipf_ids(V, B * n, seed, S_IID, step, zipf_s).reshape(B, n)
    elif kind == "uniform":
        idx = uniform_ids(V, B * n, seed, S_IID, step).reshape(B, n)
    else:
        raise ValueError(kind)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    corr = corrupt_centres(V, idx[:, n // 2], seed, step)
    return idx, corr


def scatter_inputs(rows: int, cols: int, n: int, dist: str = "zipf", payload: str = "random",
                   seed: int = 42):
    """Microbench inputs for W[I[k]] += Y[k] (BASELINE.json configs[2])."""
    if dist == "zipf":
        I = zipf_ids(rows, n, seed, S_SCATTER_I, 0)
    elif dist == "uniform":
        I = uniform_ids(rows, n, seed, S_SCATTER_I, 0)
    else:
        raise ValueError(dist)
    if payload == "random":
        Y = (2.0 * uniform01(seed, S_SCATTER_Y, 0, n * cols) - 1.0).astype(np.float32)
    elif payload == "int":
        Y = ((bits(seed, S_SCATTER_Y, 0, 0, n * cols) % np.uint64(17)).astype(np.int64) - 8).astype(np.float32)
    else:
        raise ValueError(payload)
    return I.astype(np.int32), Y.reshape(n, cols)


def random_params(V: int, d: int, n: int, h: int, seed: int, c_scale: float = 0.5,
                  w1_scale: float = None, w2_scale: float = None, b1_scale: float = 0.0,
                  b2: float = 0.0):
    """float32-representable random parameters (returned as float32 arrays).

    Defaults match the init ranges of reading G10; the *_scale knobs produce the
    saturated regime the parity tests need."""
    w1_scale = 0.5 / (n * d) if w1_scale is None else w1_scale
    w2_scale = 0.5 / h if w2_scale is None else w2_scale
    tot = V * d + n * d * h + 2 * h
    u = 2.0 * uniform01(seed, S_PARAMS, 0, tot) - 1.0
    o = 0
    C = (u[o:o + V * d] * c_scale).astype(np.float32).reshape(V, d); o += V * d
    W1 = (u[o:o + n * d * h] * w1_scale).astype(np.float32).reshape(n * d, h); o += n * d * h
    b1 = (u[o:o + h] * b1_scale).astype(np.float32); o += h
    w2 = (u[o:o + h] * w2_scale).astype(np.float32)
    return C, W1, b1, w2, np.float32(b2)


def bigram_corpus(V: int, length: int, seed: int = 42, branching: int = 4) -> np.ndarray:
    """Token stream [length] int32 of a first-order Markov chain over [0, V):
    word w's successors are succ[w][0..branching-1] (uniform draws), the next
    token is one of them, uniformly.  Consecutive windows therefore carry a
    learnable structure that a uniformly corrupted centre breaks."""
    succ = uniform_ids(V, V * branching, seed, S_BIGRAM_SUCC, 0).reshape(V, branching)
    pick = (bits(seed, S_BIGRAM_WALK, 0, 0, length) % np.uint64(branching)).astype(np.int64)
    toks = np.empty(length, np.int32)
    w = int(uniform_ids(V, 1, seed, S_BIGRAM_WALK, 1)[0])
    for i in range(length):
        toks[i] = w
        w = int(succ[w, pick[i]])
    return toks


def corpus_batch(toks: np.ndarray, V: int, n: int, B: int, seed: int, step: int, lo: int = 0, hi: int = -1):
    """B windows at i.i.d. uniform start positions in toks[lo:hi] and their
    corrupt centres (uniform, != centre)."""
    hi = toks.shape[0] if hi < 0 else hi
    starts = lo + (bits(seed, S_BIGRAM_POS, step, 0, B) % np.uint64(hi - lo - n + 1)).astype(np.int64)
    idx = np.ascontiguousarray(toks[starts[:, None] + np.arange(n)[None, :]], dtype=np.int32)
    return idx, corrupt_centres(V, idx[:, n // 2], seed, step)
