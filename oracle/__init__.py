"""SMLM oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
leg may import this package.  The product package `paper_2511_00101_b200` never imports
it and shares no code with it (no kernels, headers, helpers or constants).

* `smlm_oracle.c`  -- fp64 per-row loops of the plain SMLM definition
                      (SURVEY.md §8(c)).
* `attention.py`   -- the Alg. 1 attention branch: causal segment-wise
                      attention with KV-cache init / append, fp64 (numpy).
* `plan.py`        -- independent Python re-derivation of the canonical work plan
                      (DESIGN.md "Canonical plan").

Pinned by tests/test_oracle_pins.py (worked example, B=0, permutation, numpy dense
matmul, finite differences, special cases, linearity, Euler identities, C1 checksums).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smlm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            I = ctypes.c_int
            D = ctypes.c_double
            lib.oracle_forward.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, I, P, P, D]
            lib.oracle_forward.restype = I
            lib.oracle_backward.argtypes = [I, I, I, I, I, P, P, P, P, I, P, P, P, P, P, P, P, P, P,
                                            P, I, I, P, P, D]
            lib.oracle_backward.restype = I
            lib.oracle_num_threads.restype = I
            lib.oracle_set_num_threads.argtypes = [I]
            lib.oracle_set_num_threads.restype = None
            _lib = lib
    return _lib


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(n: int) -> None:
    """Threads of the row-parallel loops (n <= 0: all host cores); results do not depend on it."""
    _load().oracle_set_num_threads(int(n))


def _f64(t) -> np.ndarray:
    """Exact conversion of the given (bf16/fp32) values to fp64 (input rounding is not error)."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            return np.ascontiguousarray(t.detach().to("cpu", torch.float64).numpy())
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _stack(mats, shape):
    """[U, *shape] fp64.  Adapters of a smaller rank (heterogeneous ranks) are
    zero-padded to the largest rank: A_a gets zero rows, B_a zero columns.  Exact: a padded rank
    index j contributes B[:, j] (A[j] x) = 0 to y, U_j = B[:, j]^T dy = 0, so dA_a[j] = 0 and
    dB_a[:, j] = s dy (A[j] x) = 0 -- the padded entries are exact zeros and the rest is unchanged."""
    if len(mats) == 0:
        return np.zeros((1,) + shape, np.float64)
    out = np.zeros((len(mats),) + shape, np.float64)
    for i, m in enumerate(mats):
        md = _f64(m)
        out[i, :md.shape[0], :md.shape[1]] = md
    return out


def _batch_arrays(batch):
    off = np.ascontiguousarray(batch.offsets, np.int32)
    slot = np.ascontiguousarray(batch.slots, np.int32)
    mode = np.ascontiguousarray(batch.modes, np.int8)
    ss = None if batch.seg_scale is None else np.ascontiguousarray(batch.seg_scale, np.float64)
    return off, slot, mode, ss


def _keep(keep, S, in_f):
    """Dropout keep mask [S, in] (1 = kept) as uint8, or None (no dropout)."""
    if keep is None:
        return None
    k = np.ascontiguousarray(np.asarray(keep).astype(np.uint8))
    assert k.shape == (S, in_f), (k.shape, S, in_f)
    return k


def forward(batch, W, A, B, slot_scale, X, rows=None, Y_in=None, keep=None, p=0.0):
    """y_t = W x_t + s B_a (A_a x_t) in fp64.

    keep / p: LoRA dropout of FINETUNE rows (keep [S,in] bool mask, p the drop probability:
    x~ = keep * x / (1 - p) feeds A_a; smlm_oracle.c header).

    W: [out,in] or None (then Y_in [S,out] is the base output, updated in place semantics).
    A: list of [r,in]; B: list of [out,r]; slot_scale: list of floats (per slot).
    rows: optional int array of rows to compute (others left 0 / Y_in).
    Returns (Y [S,out] fp64, Vsave [S,r] fp64).
    """
    lib = _load()
    Xd = _f64(X)
    S, in_f = Xd.shape
    Wd = None if W is None else _f64(W)
    out_f = Wd.shape[0] if Wd is not None else _f64(Y_in).shape[1]
    r = max(_f64(a).shape[0] for a in A) if len(A) else 1   # largest rank (heterogeneous ranks padded)
    assert r <= 256
    Ad = _stack(A, (r, in_f))
    Bd = _stack(B, (out_f, r))
    sl = np.ascontiguousarray(np.asarray(slot_scale if len(slot_scale) else [0.0], np.float64))
    off, slot, mode, ss = _batch_arrays(batch)
    Y = np.zeros((S, out_f)) if Y_in is None else _f64(Y_in).copy()
    V = np.zeros((S, r))
    rr = None if rows is None else np.ascontiguousarray(rows, np.int64)
    kp = _keep(keep, S, in_f)
    rc = lib.oracle_forward(S, in_f, out_f, r, batch.G, _ptr(off), _ptr(slot), _ptr(mode), _ptr(ss),
                            _ptr(sl), _ptr(Ad), _ptr(Bd), _ptr(Xd), _ptr(Wd), _ptr(Y), _ptr(V),
                            0 if rr is None else len(rr), _ptr(rr), _ptr(kp), 1.0 / (1.0 - p))
    if rc != 0:
        raise ValueError("oracle_forward: malformed batch")
    return Y, V


def backward(batch, W, A, B, slot_scale, X, dY, has_grad=None, rows=None, dA_in=None, dB_in=None,
             accumulate=False, want_dx=True, keep=None, p=0.0):
    """Fine-tune backward in fp64.  Returns (dX [S,in] (zeros on non-FT rows), dA [U,r,in], dB [U,out,r]);
    r is the largest adapter rank: adapter a's gradients are dA[a, :r_a] and dB[a, :, :r_a]."""
    lib = _load()
    Xd, dYd = _f64(X), _f64(dY)
    S, in_f = Xd.shape
    out_f = dYd.shape[1]
    Wd = None if W is None else _f64(W)
    U = len(A)
    r = max(_f64(a).shape[0] for a in A) if U else 1
    Ad = _stack(A, (r, in_f))
    Bd = _stack(B, (out_f, r))
    sl = np.ascontiguousarray(np.asarray(slot_scale if U else [0.0], np.float64))
    off, slot, mode, ss = _batch_arrays(batch)
    hg = np.ones(max(U, 1), np.int32) if has_grad is None else np.ascontiguousarray(has_grad, np.int32)
    dX = np.zeros((S, in_f)) if want_dx else None
    dA = np.zeros((max(U, 1), r, in_f)) if dA_in is None else _f64(dA_in).copy()
    dB = np.zeros((max(U, 1), out_f, r)) if dB_in is None else _f64(dB_in).copy()
    rr = None if rows is None else np.ascontiguousarray(rows, np.int64)
    rc = lib.oracle_backward(S, in_f, out_f, r, batch.G, _ptr(off), _ptr(slot), _ptr(mode), _ptr(ss),
                             U, _ptr(sl), _ptr(Ad), _ptr(Bd), _ptr(Xd), _ptr(Wd), _ptr(dYd), _ptr(dX),
                             _ptr(dA), _ptr(dB), _ptr(hg), int(bool(accumulate)),
                             0 if rr is None else len(rr), _ptr(rr), _ptr(_keep(keep, S, in_f)), 1.0 / (1.0 - p))
    if rc != 0:
        raise ValueError("oracle_backward: malformed batch")
    return dX, dA[:U], dB[:U]
