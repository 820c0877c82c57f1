"""float64 CPU oracle of the Polyglot window-LM SGD step -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It shares
nothing with the CUDA product path (``paper_1404_1521_b200``): the arithmetic
lives in ``oracle/pgo.c`` (plain C, float64) and this module only marshals
numpy arrays through ctypes.

Parity pins for every function (none is "parity unpinned"):
  * pgo_forward / pgo_score  -- closed forms (zero params -> loss 1; the
    h=1 clamp case), one-hot dense brute force over a tiny
    vocabulary, swap symmetry m -> 2 - m;
  * pgo_backward             -- central finite differences of the loss in
    float64, one-hot dense form of the embedding
    gradient, saturation / inactive-hinge special cases;
  * pgo_index_add(_f32)      -- SPEC.md:67-69 worked examples, the
    10000-ones example, decomposability;
  * pgo_sgd_update           -- SPEC.md:237-238 worked examples (zero
    gradients -> unchanged; lr=1 and one sparse row -> that embedding row
    decreased by exactly the row), exact dyadic dense examples;
  * pgo_train_step(_dp)      -- theta_new == theta - lr * g with g from
    central finite differences of the loss (not pgo_backward), zero-params
    fixed point, b2 invariance, locality, DP emulation ==
    single step up to rounding;
  * tanh variant (pgo_set_activation(1)) -- finite differences (smooth, no
    kinks), the h=1 closed form s = tanh(c), zero-params fixed point;
  * sum reduction (pgo_set_reduction(1)) -- exact identities with the mean
    form (loss x B; one step at lr equals the mean step at lr x B for
    power-of-two B) and finite differences of the summed loss;
  * pgo_init_params          -- the init spec recomputed element by element
    with the independently written numpy SplitMix64 of synth/ (itself pinned
    to published SplitMix64 vectors, tests/golden/splitmix64_vectors.json),
    plus range/moment checks.
See tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_pg.so")
_SRC = os.path.join(_HERE, "pgo.c")

_lib = None


def build(force: bool = False) -> str:
    """Compile pgo.c into liboracle_pg.so with plain gcc (no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "pgo.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
             "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _SO)
    return _SO


HARDTANH, TANH = 0, 1


class activation:
    """Context manager: the oracle's nonlinearity inside the block
    (HARDTANH: north_star / reading G1; TANH: SPEC.md:70, 205), restored after."""

    _cur = HARDTANH

    def __init__(self, act):
        self.act = act

    def __enter__(self):
        self.prev = activation._cur
        if lib().pgo_set_activation(self.act) != 0:
            raise ValueError(f"unknown activation {self.act}")
        activation._cur = self.act
        return self

    def __exit__(self, *exc):
        lib().pgo_set_activation(self.prev)
        activation._cur = self.prev


MEAN, SUM = 0, 1


class reduction:
    """Context manager: batch reduction of the loss and its gradient inside the
    block (MEAN: reading G4; SUM: the summed-loss reading)."""

    _cur = MEAN

    def __init__(self, red):
        self.red = red

    def __enter__(self):
        self.prev = reduction._cur
        if lib().pgo_set_reduction(self.red) != 0:
            raise ValueError(f"unknown reduction {self.red}")
        reduction._cur = self.red
        return self

    def __exit__(self, *exc):
        lib().pgo_set_reduction(self.prev)
        reduction._cur = self.prev


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
        P = ctypes.c_void_p
        L.pgo_init_params.argtypes = [i64, i32, i32, i32, u64, P, P, P, P, P]
        L.pgo_forward.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, P, i64,
                                  P, P, P, P, P]
        L.pgo_backward.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, P, i64,
                                   ctypes.c_double, P, P, P, P, P, P, P]
        L.pgo_score.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, i64, P]
        L.pgo_train_step.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, P,
                                     i64, ctypes.c_double, P]
        L.pgo_train_step_dp.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, P,
                                        i64, i32, ctypes.c_double, P]
        L.pgo_sgd_update.argtypes = [i64, i32, i32, i32, P, P, P, P, P, ctypes.c_double,
                                     P, P, P, ctypes.c_double, P, P, i64]
        L.pgo_index_add.argtypes = [P, i64, i32, P, P, i64]
        L.pgo_index_add_f32.argtypes = [P, i64, i32, P, P, i64]
        L.pgo_last_bad.argtypes = [P, P]
        L.pgo_set_activation.argtypes = [i32]
        L.pgo_set_activation.restype = ctypes.c_int
        L.pgo_set_reduction.argtypes = [i32]
        L.pgo_set_reduction.restype = ctypes.c_int
        for f in ("pgo_init_params", "pgo_forward", "pgo_backward", "pgo_score",
                  "pgo_train_step", "pgo_train_step_dp", "pgo_index_add", "pgo_sgd_update",
                  "pgo_index_add_f32"):
            getattr(L, f).restype = ctypes.c_int
        L.pgo_last_bad.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _check(rc, what):
    if rc != 0:
        pos, val = ctypes.c_int64(), ctypes.c_int64()
        lib().pgo_last_bad(ctypes.byref(pos), ctypes.byref(val))
        extra = f" (position {pos.value}, value {val.value})" if rc == 2 else ""
        raise OracleError(rc, f"{what} failed with status {rc}{extra}")


class Params:
    """Model parameters theta = (C, W1, b1, w2, b2) in float64."""

    def __init__(self, V, d, n, h, C=None, W1=None, b1=None, w2=None, b2=0.0):
        self.V, self.d, self.n, self.h = int(V), int(d), int(n), int(h)
        self.C = np.zeros((V, d)) if C is None else np.array(C, dtype=np.float64).reshape(V, d)
        self.W1 = np.zeros((n * d, h)) if W1 is None else np.array(W1, dtype=np.float64).reshape(n * d, h)
        self.b1 = np.zeros(h) if b1 is None else np.array(b1, dtype=np.float64).reshape(h)
        self.w2 = np.zeros(h) if w2 is None else np.array(w2, dtype=np.float64).reshape(h)
        self.b2 = np.array([float(b2)], dtype=np.float64)

    @classmethod
    def init(cls, V, d, n, h, seed):
        p = cls(V, d, n, h)
        _check(lib().pgo_init_params(V, d, n, h, seed, _p(p.C), _p(p.W1), _p(p.b1),
                                     _p(p.w2), _p(p.b2)), "pgo_init_params")
        return p

    def copy(self):
        return Params(self.V, self.d, self.n, self.h, self.C.copy(), self.W1.copy(),
                      self.b1.copy(), self.w2.copy(), float(self.b2[0]))

    def _args(self):
        return (self.V, self.d, self.n, self.h, _p(self.C), _p(self.W1), _p(self.b1),
                _p(self.w2), _p(self.b2))

    def flat(self):
        return np.concatenate([self.C.ravel(), self.W1.ravel(), self.b1, self.w2, self.b2])


def forward(p: Params, idx, corr):
    idx, corr = _i32(idx), _i32(corr)
    B = corr.shape[0]
    a = np.zeros((B, p.h)); ac = np.zeros((B, p.h))
    s = np.zeros(B); sc = np.zeros(B); loss = np.zeros(1)
    _check(lib().pgo_forward(*p._args(), _p(idx), _p(corr), B, _p(a), _p(ac), _p(s),
                             _p(sc), _p(loss)), "pgo_forward")
    return dict(a=a, a_corr=ac, s=s, s_corr=sc, loss=float(loss[0]))


def loss(p: Params, idx, corr) -> float:
    idx, corr = _i32(idx), _i32(corr)
    out = np.zeros(1)
    _check(lib().pgo_forward(*p._args(), _p(idx), _p(corr), corr.shape[0], None, None,
                             None, None, _p(out)), "pgo_forward")
    return float(out[0])


def backward(p: Params, idx, corr, inv_batch=None):
    idx, corr = _i32(idx), _i32(corr)
    B = corr.shape[0]
    inv = (1.0 if reduction._cur == SUM else 1.0 / B) if inv_batch is None else float(inv_batch)
    dW1 = np.zeros_like(p.W1); db1 = np.zeros(p.h); dw2 = np.zeros(p.h); db2 = np.zeros(1)
    rows = np.zeros(2 * p.n * B, dtype=np.int32)
    Y = np.zeros((2 * p.n * B, p.d))
    nrows = ctypes.c_int64()
    _check(lib().pgo_backward(*p._args(), _p(idx), _p(corr), B, inv, _p(dW1), _p(db1),
                              _p(dw2), _p(db2), _p(rows), _p(Y), ctypes.byref(nrows)),
           "pgo_backward")
    r = nrows.value
    return dict(dW1=dW1, db1=db1, dw2=dw2, db2=float(db2[0]), rows=rows[:r], Y=Y[:r])


def score(p: Params, idx):
    idx = _i32(idx)
    B = idx.shape[0]
    out = np.zeros(B)
    _check(lib().pgo_score(*p._args(), _p(idx), B, _p(out)), "pgo_score")
    return out


def sgd_update(p: Params, grads: dict, lr) -> None:
    """In-place SPEC.md:231-235 update: dense theta -= lr * grad, C by the serial
    index_add of -lr * Y over grads["rows"]."""
    h, nd = p.h, p.n * p.d
    dW1 = np.ascontiguousarray(grads.get("dW1", np.zeros((nd, h))), np.float64)
    db1 = np.ascontiguousarray(grads.get("db1", np.zeros(h)), np.float64)
    dw2 = np.ascontiguousarray(grads.get("dw2", np.zeros(h)), np.float64)
    rows = _i32(grads.get("rows", np.zeros(0, np.int32)))
    Y = np.ascontiguousarray(grads.get("Y", np.zeros((0, p.d))), np.float64).reshape(-1, p.d)
    if Y.shape[0] != rows.shape[0]:
        raise ValueError("Y and rows disagree")
    _check(lib().pgo_sgd_update(*p._args(), float(lr), _p(dW1), _p(db1), _p(dw2),
                                float(grads.get("db2", 0.0)), _p(rows), _p(Y), rows.shape[0]),
           "pgo_sgd_update")


def train_step(p: Params, idx, corr, lr) -> float:
    """In-place SGD step on p; returns the pre-update mean loss."""
    idx, corr = _i32(idx), _i32(corr)
    out = np.zeros(1)
    _check(lib().pgo_train_step(*p._args(), _p(idx), _p(corr), corr.shape[0], float(lr),
                                _p(out)), "pgo_train_step")
    return float(out[0])


def train_step_dp(p: Params, idx, corr, lr, world) -> float:
    idx, corr = _i32(idx), _i32(corr)
    out = np.zeros(1)
    _check(lib().pgo_train_step_dp(*p._args(), _p(idx), _p(corr), corr.shape[0],
                                   int(world), float(lr), _p(out)), "pgo_train_step_dp")
    return float(out[0])


def index_add(W, Y, I):
    """Serial W[I[k]] += Y[k] for k in order; W mutated in place."""
    I = _i32(I)
    if W.dtype == np.float32:
        Y = np.ascontiguousarray(Y, dtype=np.float32)
        _check(lib().pgo_index_add_f32(_p(W), W.shape[0], W.shape[1], _p(Y), _p(I),
                                       I.shape[0]), "pgo_index_add_f32")
    else:
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        _check(lib().pgo_index_add(_p(W), W.shape[0], W.shape[1], _p(Y), _p(I),
                                   I.shape[0]), "pgo_index_add")
    return W
