"""Python binding of libpg (include/pg.h): argument marshalling only.

Every step of the SGD step and of the scatter-add runs in the sm_100a kernels
of ``libpg.so``; this module only converts tensors/arrays to pointers and
status codes to exceptions.  There is no CPU fallback: importing succeeds
without a GPU (so the ABI can be inspected), but every compute call needs the
built library and a CUDA device and raises otherwise.

Names follow the C ABI: pg_init, pg_train_step, pg_score, pg_free,
pg_get_params, pg_set_params, pg_set_option, pg_sync, pg_scatter_add,
pg_nccl_unique_id, pg_attach_nccl.  ``PolyglotModel`` is a convenience holder
for the opaque handle.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PG_LIB_VARIANT=trace selects the instrumented build (libpg_trace.so, see build.py)
LIB_PATH = os.path.join(_HERE, "libpg_trace.so" if os.environ.get("PG_LIB_VARIANT") == "trace" else "libpg.so")
# PG_LIB_PATH overrides it (A/B experiments: scripts/ab_variant.py builds variant libraries)
LIB_PATH = os.environ.get("PG_LIB_PATH", LIB_PATH)

PG_OK, PG_EINVAL, PG_ERANGE, PG_ENOMEM, PG_ECUDA, PG_ENCCL, PG_EDIVERGED = range(7)
PG_SCATTER_DET, PG_SCATTER_ATOMIC = 0, 1
PG_OPT_SCATTER, PG_OPT_STREAM, PG_OPT_FUSED, PG_OPT_RESERVE, PG_OPT_TRACE, PG_OPT_ACTIVATION = 1, 2, 3, 4, 5, 6
PG_OPT_REDUCTION = 7
PG_OPT_EXCHANGE = 8
PG_EXCHANGE_AUTO, PG_EXCHANGE_PEER, PG_EXCHANGE_ALLGATHER, PG_EXCHANGE_TABLE = 0, 1, 2, 3
EXCHANGE_NAMES = {-1: "none", 0: "auto", 1: "peer", 2: "allgather", 3: "table"}
PG_ACT_HARDTANH, PG_ACT_TANH = 0, 1
PG_REDUCE_MEAN, PG_REDUCE_SUM = 0, 1

EXPORTED = [
    "pg_init", "pg_train_step", "pg_train_step_loss", "pg_score", "pg_free", "pg_last_error",
    "pg_get_params", "pg_set_params", "pg_get_shape", "pg_set_option", "pg_sync",
    "pg_scatter_add", "pg_scatter_add_async", "pg_nccl_unique_id", "pg_attach_nccl",
    "pg_kernel_launches", "pg_abi_version", "pg_train_step_group", "pg_exchange_info",
]

_lib = None


class PGError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[pg status {status}] {msg}")
        self.status = status


def lib():
    """Load libpg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1404_1521_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        sig = {
            "pg_init": ([ctypes.POINTER(P), i64, i32, i32, i32, ctypes.c_uint64], ctypes.c_int),
            "pg_train_step": ([P, P, P, i32, f32, P], ctypes.c_int),
            "pg_train_step_loss": ([P, P, P, i32, f32], f32),
            "pg_score": ([P, P, i32, P], ctypes.c_int),
            "pg_free": ([P], None),
            "pg_last_error": ([], ctypes.c_char_p),
            "pg_get_params": ([P, P, P, P, P, P], ctypes.c_int),
            "pg_set_params": ([P, P, P, P, P, f32], ctypes.c_int),
            "pg_get_shape": ([P, P, P, P, P], ctypes.c_int),
            "pg_set_option": ([P, ctypes.c_int, i64], ctypes.c_int),
            "pg_sync": ([P], ctypes.c_int),
            "pg_scatter_add": ([P, i64, i32, P, P, i64, ctypes.c_int, P], ctypes.c_int),
            "pg_scatter_add_async": ([P, i64, i32, P, P, i64, ctypes.c_int, P, P], ctypes.c_int),
            "pg_nccl_unique_id": ([P], ctypes.c_int),
            "pg_attach_nccl": ([P, ctypes.c_int, ctypes.c_int, P], ctypes.c_int),
            "pg_kernel_launches": ([P], i64),
            "pg_abi_version": ([], ctypes.c_int),
            "pg_train_step_group": ([P, ctypes.c_int, P, P, i32, f32, P], ctypes.c_int),
            "pg_exchange_info": ([P, P, P, ctypes.c_int], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def pg_last_error() -> str:
    return lib().pg_last_error().decode()


def _check(rc, what):
    if rc != PG_OK:
        raise PGError(rc, f"{what}: {pg_last_error()}")


_TDT = {}


def _torch_dtype(dtype):
    t = _TDT.get(dtype)
    if t is None:
        import torch
        t = _TDT[dtype] = {np.int32: torch.int32, np.float32: torch.float32}[dtype]
    return t


def _ptr(x, dtype=None):
    """Pointer of a torch tensor (any device) or numpy array; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        if dtype is not None and x.dtype != dtype:
            raise TypeError(f"expected {dtype}, got {x.dtype}")
        return ctypes.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if dtype is not None:
            tdt = _torch_dtype(dtype)
            if x.dtype != tdt:
                raise TypeError(f"expected {tdt}, got {x.dtype}")
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    raise TypeError(f"unsupported argument type {type(x)}")


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ---------------------------------------------------------------------- C-ABI mirrors
def pg_init(vocab, dim, window, hidden, seed=42):
    h = ctypes.c_void_p()
    _check(lib().pg_init(ctypes.byref(h), int(vocab), int(dim), int(window), int(hidden),
                         int(seed) & 0xFFFFFFFFFFFFFFFF), "pg_init")
    _SHAPES[_hkey(h)] = int(window)
    return h


def pg_free(handle):
    _SHAPES.pop(_hkey(handle), None)
    lib().pg_free(handle)


def pg_set_option(handle, key, value):
    _check(lib().pg_set_option(handle, int(key), int(value)), "pg_set_option")


_HOST = "host"


def _window_of(handle):
    n = _SHAPES.get(_hkey(handle))
    if n is None:
        n = pg_get_shape(handle)[2]
    return n


def _hkey(handle):
    return handle.value if hasattr(handle, "value") else int(handle)


_SHAPES = {}   # handle -> window (cached by pg_init; pg_get_shape otherwise)


def _check_batch(handle, idx_batch, corrupt_idx=None):
    """The C side reads batch*window ints of idx and batch of corr: mismatched
    arrays would be out-of-bounds reads, so reject them here (ValueError)."""
    n = _window_of(handle)
    if len(idx_batch.shape) == 2:
        if int(idx_batch.shape[1]) != n:
            raise ValueError(f"idx_batch has {idx_batch.shape[1]} columns, the model window is {n}")
        batch = int(idx_batch.shape[0])
    elif len(idx_batch.shape) == 1:
        if int(idx_batch.shape[0]) % n:
            raise ValueError(f"flat idx_batch of {idx_batch.shape[0]} ints is not a multiple of window {n}")
        batch = int(idx_batch.shape[0]) // n
    else:
        raise ValueError("idx_batch must be [batch][window] (or flat batch*window)")
    if corrupt_idx is not None:
        if len(corrupt_idx.shape) != 1 or int(corrupt_idx.shape[0]) != batch:
            raise ValueError(f"corrupt_idx must have shape ({batch},), got {tuple(corrupt_idx.shape)}")
    return batch


def pg_train_step(handle, idx_batch, corrupt_idx, lr, loss_out=_HOST):
    """One SGD step.  loss_out="host" -> blocking, returns the float loss;
    a device or pinned-host float32 tensor -> asynchronous, the step kernel
    writes the loss there; None -> async (include/pg.h)."""
    batch = _check_batch(handle, idx_batch, corrupt_idx)
    # `is`, not `==`: comparing a torch tensor with a str costs ~13 us per call
    if loss_out is _HOST or (isinstance(loss_out, str) and loss_out == "host"):
        out = ctypes.c_float()
        _check(lib().pg_train_step(handle, _ptr(idx_batch, np.int32), _ptr(corrupt_idx, np.int32),
                                   batch, float(lr), ctypes.cast(ctypes.byref(out), ctypes.c_void_p)),
               "pg_train_step")
        return out.value
    _check(lib().pg_train_step(handle, _ptr(idx_batch, np.int32), _ptr(corrupt_idx, np.int32), batch,
                               float(lr), _ptr(loss_out, np.float32)), "pg_train_step")
    return None


def pg_train_step_loss(handle, idx_batch, corrupt_idx, lr):
    batch = _check_batch(handle, idx_batch, corrupt_idx)
    return lib().pg_train_step_loss(handle, _ptr(idx_batch, np.int32), _ptr(corrupt_idx, np.int32),
                                    batch, float(lr))


def pg_score(handle, idx_batch, scores_out=None):
    batch = _check_batch(handle, idx_batch)
    if scores_out is None:
        scores_out = np.zeros(batch, np.float32)
    if len(scores_out.shape) != 1 or int(scores_out.shape[0]) < batch:
        raise ValueError(f"scores_out must hold {batch} floats")
    _check(lib().pg_score(handle, _ptr(idx_batch, np.int32), batch, _ptr(scores_out, np.float32)),
           "pg_score")
    return scores_out


def pg_get_shape(handle):
    V, d, n, h = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().pg_get_shape(handle, ctypes.byref(V), ctypes.byref(d), ctypes.byref(n),
                              ctypes.byref(h)), "pg_get_shape")
    return V.value, d.value, n.value, h.value


def pg_get_params(handle):
    """(C, W1, b1, w2, b2) as float32 numpy arrays in the canonical layouts."""
    V, d, n, h = pg_get_shape(handle)
    C = np.empty((V, d), np.float32); W1 = np.empty((n * d, h), np.float32)
    b1 = np.empty(h, np.float32); w2 = np.empty(h, np.float32); b2 = np.empty(1, np.float32)
    _check(lib().pg_get_params(handle, _ptr(C), _ptr(W1), _ptr(b1), _ptr(w2), _ptr(b2)),
           "pg_get_params")
    return C, W1, b1, w2, float(b2[0])


def pg_set_params(handle, C=None, W1=None, b1=None, w2=None, b2=None):
    def prep(a):
        if a is None or hasattr(a, "data_ptr"):
            return a
        return np.ascontiguousarray(a, dtype=np.float32)
    C, W1, b1, w2 = prep(C), prep(W1), prep(b1), prep(w2)
    _check(lib().pg_set_params(handle, _ptr(C), _ptr(W1), _ptr(b1), _ptr(w2),
                               float("nan") if b2 is None else float(b2)), "pg_set_params")


def pg_sync(handle):
    _check(lib().pg_sync(handle), "pg_sync")


def pg_scatter_add(W, Y, I, mode=PG_SCATTER_DET, stream=None, blocking=True, err_flag=None):
    """W[I[k], :] += Y[k, :] on device tensors."""
    if len(W.shape) != 2:
        raise ValueError("W must be 2-D [rows][cols]")
    if len(I.shape) != 1:
        raise ValueError("I must be 1-D")
    n = int(I.shape[0])
    rows, cols = int(W.shape[0]), int(W.shape[1])
    if tuple(Y.shape) != (n, cols) and not (n == 0 and int(np.prod(Y.shape)) == 0):
        raise ValueError(f"Y must have shape ({n}, {cols}), got {tuple(Y.shape)}")
    s = ctypes.c_void_p(_stream_handle(stream))
    if blocking:
        _check(lib().pg_scatter_add(_ptr(W, np.float32), rows, cols, _ptr(Y, np.float32),
                                    _ptr(I, np.int32), n, int(mode), s), "pg_scatter_add")
    else:
        _check(lib().pg_scatter_add_async(_ptr(W, np.float32), rows, cols, _ptr(Y, np.float32),
                                          _ptr(I, np.int32), n, int(mode), s, _ptr(err_flag)),
               "pg_scatter_add_async")
    return W


def pg_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().pg_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "pg_nccl_unique_id")
    return buf.raw


def pg_attach_nccl(handle, rank, world, unique_id: bytes):
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(lib().pg_attach_nccl(handle, int(rank), int(world), ctypes.cast(buf, ctypes.c_void_p)),
           "pg_attach_nccl")


def pg_exchange_info(handle, reset=False):
    """(exchange in use as a name, bytes read from other ranks, max entries one
    owner merged) since the last reset."""
    mode = ctypes.c_int()
    st = (ctypes.c_uint64 * 2)()
    _check(lib().pg_exchange_info(handle, ctypes.byref(mode), ctypes.cast(st, ctypes.c_void_p), int(bool(reset))),
           "pg_exchange_info")
    return EXCHANGE_NAMES.get(mode.value, str(mode.value)), int(st[0]), int(st[1])


def pg_kernel_launches(handle) -> int:
    return int(lib().pg_kernel_launches(handle))


# ---------------------------------------------------------------------- convenience holder
class PolyglotModel:
    """Owns a pg_model handle; methods forward to the C ABI with the torch stream."""

    def __init__(self, vocab, dim, window, hidden, seed=42, scatter=PG_SCATTER_DET, stream=None,
                 fused=True, activation=PG_ACT_HARDTANH, reduction=PG_REDUCE_MEAN, exchange=PG_EXCHANGE_AUTO):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("PolyglotModel needs a CUDA device (no CPU fallback)")
        self.handle = pg_init(vocab, dim, window, hidden, seed)
        self.shape = (vocab, dim, window, hidden)
        pg_set_option(self.handle, PG_OPT_STREAM, _stream_handle(stream))
        pg_set_option(self.handle, PG_OPT_SCATTER, scatter)
        pg_set_option(self.handle, PG_OPT_FUSED, 1 if fused else 0)
        pg_set_option(self.handle, PG_OPT_ACTIVATION, activation)
        pg_set_option(self.handle, PG_OPT_REDUCTION, reduction)
        pg_set_option(self.handle, PG_OPT_EXCHANGE, exchange)

    def set_stream(self, stream):
        pg_set_option(self.handle, PG_OPT_STREAM, _stream_handle(stream))

    def reserve(self, batch):
        pg_set_option(self.handle, PG_OPT_RESERVE, batch)

    def train_step(self, idx, corr, lr, loss_out="host"):
        return pg_train_step(self.handle, idx, corr, lr, loss_out)

    def score(self, idx, out=None):
        return pg_score(self.handle, idx, out)

    def get_params(self):
        return pg_get_params(self.handle)

    def set_params(self, C=None, W1=None, b1=None, w2=None, b2=None):
        pg_set_params(self.handle, C, W1, b1, w2, b2)

    def sync(self):
        pg_sync(self.handle)

    def attach_nccl(self, rank, world, uid):
        pg_attach_nccl(self.handle, rank, world, uid)

    def exchange_info(self, reset=False):
        return pg_exchange_info(self.handle, reset)

    def kernel_launches(self):
        return pg_kernel_launches(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            pg_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pg_abi_version() -> int:
    return int(lib().pg_abi_version())


def pg_scatter_add_async(W, Y, I, mode=PG_SCATTER_DET, stream=None, err_flag=None):
    return pg_scatter_add(W, Y, I, mode, stream, blocking=False, err_flag=err_flag)


def pg_train_step_group(handles, idx_all, corr_all, lr):
    """One data-parallel step of len(handles) replicas on one device (contiguous
    shards of idx_all / corr_all); returns the global mean loss."""
    world = len(handles)
    arr = (ctypes.c_void_p * world)(*[h.value if hasattr(h, "value") else h for h in handles])
    if int(corr_all.shape[0]) % world:
        raise ValueError(f"global batch {corr_all.shape[0]} is not divisible by {world} replicas")
    _check_batch(handles[0], idx_all, corr_all)
    batch_local = int(corr_all.shape[0]) // world
    out = ctypes.c_float()
    _check(lib().pg_train_step_group(ctypes.cast(arr, ctypes.c_void_p), world, _ptr(idx_all, np.int32),
                                     _ptr(corr_all, np.int32), batch_local, float(lr),
                                     ctypes.cast(ctypes.byref(out), ctypes.c_void_p)), "pg_train_step_group")
    return out.value
