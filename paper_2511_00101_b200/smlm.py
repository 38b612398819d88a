"""Thin ctypes binding of libsmlm.so (include/smlm.h).  Argument marshalling only: every step
of the SMLM path runs in the library's CUDA kernels.  PyTorch supplies device memory and streams.

Function names mirror the C ABI (smlm_pool_create, smlm_adapter_register, smlm_forward, ...);
`Pool` is a convenience owner that keeps borrowed adapter tensors alive.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# the release library; SMLM_MEASURE_LIB=1 loads the -DSMLM_MEASURE build (build.py --measure:
# phase timestamps / host timing for the scripts under scripts/, same kernels and results);
# SMLM_LIB_PATH loads another build of the same C ABI (same-box A/B of two library versions)
LIB_PATH = os.environ.get("SMLM_LIB_PATH") or os.path.join(
    _HERE, "libsmlm_measure.so" if os.environ.get("SMLM_MEASURE_LIB") == "1" else "libsmlm.so")

SMLM_OK, SMLM_E_INVALID, SMLM_E_SHAPE, SMLM_E_SLOT, SMLM_E_CAPACITY, SMLM_E_CUDA, SMLM_E_UNSUPPORTED, \
    SMLM_E_WORKSPACE = range(8)
SMLM_FINETUNE, SMLM_EVAL, SMLM_PREFILL, SMLM_DECODE = range(4)
SMLM_BF16, SMLM_FP32 = 0, 1
SMLM_OPT_L_LONG, SMLM_OPT_CTA_PAIR, SMLM_OPT_DECODE_KERNEL, SMLM_OPT_DEC_KSPLIT, SMLM_OPT_DEC_COOPERATIVE = 0, 1, 2, 3, 4
PROF_FWD_GEMM, PROF_BWD_GEMM, PROF_SHRINK, PROF_DADB, PROF_ADAMW = range(5)

EXPORTED = [
    "smlm_pool_create", "smlm_pool_destroy", "smlm_pool_set_option", "smlm_adapter_register",
    "smlm_adapter_set_grad", "smlm_adapter_unregister", "smlm_workspace_size", "smlm_forward",
    "smlm_backward", "smlm_plan", "smlm_plan_export", "smlm_status_string", "smlm_last_error",
    "smlm_launch_count", "smlm_profile_enable", "smlm_profile_read", "smlm_workspace_size_multi",
    "smlm_forward_multi", "smlm_adamw_workspace_size", "smlm_adamw_step", "smlm_adapter_register_rank",
    "smlm_workspace_size_backward_multi", "smlm_backward_multi",
    "smlm_ipc_get_handle", "smlm_ipc_open_handle", "smlm_ipc_close_handle", "smlm_pool_set_grad_fanout",
    "smlm_fanout_signal", "smlm_fanout_wait", "smlm_adamw_step_reduce",
    "smlm_attention_workspace_size", "smlm_attention",
]


class SmlmError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {_status_name(code)}: {msg}")
        self.code = code


class smlm_batch(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int), ("G", ctypes.c_int), ("seg_offsets", ctypes.c_void_p),
                ("seg_slot", ctypes.c_void_p), ("seg_mode", ctypes.c_void_p), ("seg_scale", ctypes.c_void_p),
                ("dropout_p", ctypes.c_float), ("dropout_seed", ctypes.c_uint64)]


class smlm_attn_batch(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int), ("G", ctypes.c_int), ("seg_offsets", ctypes.c_void_p),
                ("seg_mode", ctypes.c_void_p), ("seg_cache", ctypes.c_void_p), ("seg_past", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsmlm.so not built at {LIB_PATH}: run `python -m paper_2511_00101_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    BP = ctypes.POINTER(smlm_batch)
    sig = {
        "smlm_pool_create": ([I, I, I, I, I, I, ctypes.POINTER(P)], I),
        "smlm_pool_destroy": ([P], I),
        "smlm_pool_set_option": ([P, I, I], I),
        "smlm_adapter_register": ([P, P, P, ctypes.c_float, P, ctypes.POINTER(I)], I),
        "smlm_adapter_register_rank": ([P, P, P, I, ctypes.c_float, P, ctypes.POINTER(I)], I),
        "smlm_adapter_set_grad": ([P, I, P, P], I),
        "smlm_adapter_unregister": ([P, I, P], I),
        "smlm_workspace_size": ([P, BP, I], Z),
        "smlm_forward": ([P, BP, P, P, P, P, P, Z, P], I),
        "smlm_workspace_size_multi": ([I, P, BP], Z),
        "smlm_forward_multi": ([I, P, BP, P, P, P, P, P, Z, P], I),
        "smlm_backward": ([P, BP, P, P, P, P, P, I, P, Z, P], I),
        "smlm_workspace_size_backward_multi": ([I, P, BP], Z),
        "smlm_backward_multi": ([I, P, BP, P, P, P, P, P, I, P, Z, P], I),
        "smlm_plan": ([BP, I, P, I, I, P, I, ctypes.POINTER(I)], I),
        "smlm_plan_export": ([P, BP, I, P, I, ctypes.POINTER(I)], I),
        "smlm_status_string": ([I], ctypes.c_char_p),
        "smlm_last_error": ([], ctypes.c_char_p),
        "smlm_launch_count": ([], ctypes.c_uint64),
        "smlm_profile_enable": ([I], I),
        "smlm_profile_read": ([I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I)], I),
        "smlm_adamw_workspace_size": ([], Z),
        "smlm_adamw_step": ([P, P, P, P, P, Z, I] + [ctypes.c_float] * 7 + [I, P, Z, P], I),
        "smlm_adamw_step_reduce": ([P, P, P, P, I, Z, I, P, Z, I] + [ctypes.c_float] * 7 + [I, P, I, P, Z, P], I),
        "smlm_ipc_get_handle": ([P, P, ctypes.POINTER(ctypes.c_uint64)], I),
        "smlm_ipc_open_handle": ([P, ctypes.POINTER(P)], I),
        "smlm_ipc_close_handle": ([P], I),
        "smlm_pool_set_grad_fanout": ([P, I, P], I),
        "smlm_fanout_signal": ([I, P, P], I),
        "smlm_fanout_wait": ([P, I, P], I),
        "smlm_attention_workspace_size": ([ctypes.POINTER(smlm_attn_batch), I, I], Z),
        "smlm_attention": ([ctypes.POINTER(smlm_attn_batch), I, I, I, P, P, P, P, P, P, I, I, ctypes.c_float, P, Z, P],
                           I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()


def _status_name(code: int) -> str:
    return _lib.smlm_status_string(code).decode()


def _check(code: int, where: str):
    if code != SMLM_OK:
        raise SmlmError(code, where, _lib.smlm_last_error().decode())


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream, device) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Batch:
    """Host-side segment arrays kept alive for the duration of the calls."""

    def __init__(self, offsets, slots, modes, seg_scale=None, dropout_p=0.0, dropout_seed=0):
        self.offsets = np.ascontiguousarray(offsets, np.int32)
        self.slots = np.ascontiguousarray(slots, np.int32)
        self.modes = np.ascontiguousarray(modes, np.int8)
        self.seg_scale = None if seg_scale is None else np.ascontiguousarray(seg_scale, np.float32)
        self.c = smlm_batch(int(self.offsets[-1]) if len(self.offsets) else 0, len(self.slots),
                            self.offsets.ctypes.data, self.slots.ctypes.data, self.modes.ctypes.data,
                            None if self.seg_scale is None else self.seg_scale.ctypes.data,
                            float(dropout_p), int(dropout_seed) & 0xFFFFFFFFFFFFFFFF)

    def with_dropout(self, p: float, seed: int) -> "Batch":
        """The same segments with LoRA dropout p on the fine-tune rows and mask seed `seed`."""
        return Batch(self.offsets, self.slots, self.modes, self.seg_scale, p, seed)

    @classmethod
    def from_synth(cls, b, dropout_p=0.0, dropout_seed=0):
        return cls(b.offsets, b.slots, b.modes, b.seg_scale, dropout_p, dropout_seed)

    @property
    def S(self):
        return self.c.S


# ------------------------------ C-ABI mirrors ------------------------------
def smlm_pool_create(device: int, in_features: int, out_features: int, rank: int, capacity: int,
                     dtype: int = SMLM_BF16) -> int:
    h = ctypes.c_void_p()
    _check(_lib.smlm_pool_create(device, in_features, out_features, rank, capacity, dtype, ctypes.byref(h)),
           "smlm_pool_create")
    return h.value


def smlm_pool_destroy(pool: int):
    _check(_lib.smlm_pool_destroy(pool), "smlm_pool_destroy")


def smlm_pool_set_option(pool: int, option: int, value: int):
    _check(_lib.smlm_pool_set_option(pool, option, value), "smlm_pool_set_option")


def smlm_adapter_register(pool: int, A, B, scale: float, stream=None) -> int:
    s = ctypes.c_int(-1)
    _check(_lib.smlm_adapter_register(pool, _ptr(A), _ptr(B), float(scale), _stream(stream, A.device),
                                      ctypes.byref(s)), "smlm_adapter_register")
    return s.value


def smlm_adapter_register_rank(pool: int, A, B, rank: int, scale: float, stream=None) -> int:
    s = ctypes.c_int(-1)
    _check(_lib.smlm_adapter_register_rank(pool, _ptr(A), _ptr(B), int(rank), float(scale),
                                           _stream(stream, A.device), ctypes.byref(s)), "smlm_adapter_register_rank")
    return s.value


def smlm_adapter_set_grad(pool: int, slot: int, dA=None, dB=None):
    _check(_lib.smlm_adapter_set_grad(pool, slot, _ptr(dA), _ptr(dB)), "smlm_adapter_set_grad")


def smlm_adapter_unregister(pool: int, slot: int, stream=None, device=None):
    _check(_lib.smlm_adapter_unregister(pool, slot, _stream(stream, device)), "smlm_adapter_unregister")


def smlm_workspace_size(pool: int, batch: Batch, backward: bool) -> int:
    return int(_lib.smlm_workspace_size(pool, ctypes.byref(batch.c), int(backward)))


def smlm_forward(pool: int, batch: Batch, X, W, Y, V_save=None, ws=None, stream=None):
    _check(_lib.smlm_forward(pool, ctypes.byref(batch.c), _ptr(X), _ptr(W), _ptr(Y), _ptr(V_save), _ptr(ws),
                             0 if ws is None else ws.numel() * ws.element_size(), _stream(stream, X.device)),
           "smlm_forward")


def _ptr_array(xs):
    arr = (ctypes.c_void_p * len(xs))(*[None if x is None else (x if isinstance(x, int) else x.data_ptr())
                                        for x in xs])
    return arr


def smlm_workspace_size_multi(pools, batch: Batch) -> int:
    hs = _ptr_array(list(pools))
    return int(_lib.smlm_workspace_size_multi(len(pools), ctypes.cast(hs, ctypes.c_void_p), ctypes.byref(batch.c)))


def smlm_forward_multi(pools, batch: Batch, X, Ws, Ys, V_saves=None, ws=None, stream=None):
    """One call for several projections sharing X (q/k/v, gate/up): include/smlm.h smlm_forward_multi."""
    n = len(pools)
    hs, wp, yp = _ptr_array(list(pools)), _ptr_array(Ws), _ptr_array(Ys)
    vp = None if V_saves is None else _ptr_array(V_saves)
    _check(_lib.smlm_forward_multi(n, ctypes.cast(hs, ctypes.c_void_p), ctypes.byref(batch.c), _ptr(X),
                                   ctypes.cast(wp, ctypes.c_void_p), ctypes.cast(yp, ctypes.c_void_p),
                                   None if vp is None else ctypes.cast(vp, ctypes.c_void_p), _ptr(ws),
                                   0 if ws is None else ws.numel() * ws.element_size(), _stream(stream, X.device)),
           "smlm_forward_multi")


def smlm_backward(pool: int, batch: Batch, X, W, dY, V_save=None, dX=None, accumulate=False, ws=None,
                  stream=None):
    _check(_lib.smlm_backward(pool, ctypes.byref(batch.c), _ptr(X), _ptr(W), _ptr(dY), _ptr(V_save), _ptr(dX),
                              int(bool(accumulate)), _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                              _stream(stream, X.device)), "smlm_backward")


def smlm_workspace_size_backward_multi(pools, batch: Batch) -> int:
    hs = _ptr_array(list(pools))
    return int(_lib.smlm_workspace_size_backward_multi(len(pools), ctypes.cast(hs, ctypes.c_void_p),
                                                       ctypes.byref(batch.c)))


def smlm_backward_multi(pools, batch: Batch, X, Ws, dYs, V_saves, dXs, accumulate=False, ws=None, stream=None):
    """Backward of several projections sharing X (include/smlm.h smlm_backward_multi)."""
    n = len(pools)
    hs, wp, yp, xp = _ptr_array(list(pools)), _ptr_array(Ws), _ptr_array(dYs), _ptr_array(dXs)
    vp = None if V_saves is None else _ptr_array(V_saves)
    c = lambda a: ctypes.cast(a, ctypes.c_void_p)  # noqa: E731
    _check(_lib.smlm_backward_multi(n, c(hs), ctypes.byref(batch.c), _ptr(X), c(wp), c(yp),
                                    None if vp is None else c(vp), c(xp), int(bool(accumulate)), _ptr(ws),
                                    0 if ws is None else ws.numel() * ws.element_size(), _stream(stream, X.device)),
           "smlm_backward_multi")


def smlm_plan(batch: Batch, capacity: int, registered, l_long: int = 64, backward: bool = False):
    reg = np.ascontiguousarray(registered, np.uint8)
    n = ctypes.c_int(0)
    code = _lib.smlm_plan(ctypes.byref(batch.c), capacity, reg.ctypes.data, l_long, int(backward), None, 0,
                          ctypes.byref(n))
    if code not in (SMLM_OK, SMLM_E_WORKSPACE):
        _check(code, "smlm_plan")
    buf = np.zeros((max(n.value, 1), 6), np.int32)
    _check(_lib.smlm_plan(ctypes.byref(batch.c), capacity, reg.ctypes.data, l_long, int(backward),
                          buf.ctypes.data, n.value, ctypes.byref(n)), "smlm_plan")
    return buf[:n.value].tolist()


def smlm_plan_export(pool: int, batch: Batch, backward: bool = False):
    n = ctypes.c_int(0)
    code = _lib.smlm_plan_export(pool, ctypes.byref(batch.c), int(backward), None, 0, ctypes.byref(n))
    if code not in (SMLM_OK, SMLM_E_WORKSPACE):
        _check(code, "smlm_plan_export")
    buf = np.zeros((max(n.value, 1), 6), np.int32)
    _check(_lib.smlm_plan_export(pool, ctypes.byref(batch.c), int(backward), buf.ctypes.data, n.value,
                                 ctypes.byref(n)), "smlm_plan_export")
    return buf[:n.value].tolist()


def smlm_adamw_workspace_size() -> int:
    return int(_lib.smlm_adamw_workspace_size())


def smlm_adamw_step(param, exp_avg, exp_avg_sq, grad, param_bf16, step: int, lr: float, beta1: float = 0.9,
                    beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0, grad_scale: float = 1.0,
                    max_grad_norm: float = 0.0, zero_grad: bool = False, ws=None, stream=None):
    """AdamW over flat fp32 buffers of n elements (include/smlm.h smlm_adamw_step)."""
    n = param.numel()
    for t in (exp_avg, exp_avg_sq, grad) + (() if param_bf16 is None else (param_bf16,)):
        if t.numel() != n:
            raise ValueError("smlm_adamw_step: every buffer must have param.numel() elements")
    _check(_lib.smlm_adamw_step(_ptr(param), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad), _ptr(param_bf16), n,
                                int(step), lr, beta1, beta2, eps, weight_decay, grad_scale, max_grad_norm,
                                int(bool(zero_grad)), _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                                _stream(stream, param.device)), "smlm_adamw_step")


def smlm_adamw_step_reduce(param, exp_avg, exp_avg_sq, grad_slots, n_slots: int, slot_stride: int, own_slot: int,
                           param_bf16, n: int, step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
                           eps: float = 1e-8, weight_decay: float = 0.0, grad_scale: float = 1.0,
                           max_grad_norm: float = 0.0, zero_grad: bool = False, ready=None, ready_target: int = 0,
                           ws=None, stream=None):
    """AdamW on the rank-ordered sum of n_slots gradient slots (include/smlm.h smlm_adamw_step_reduce).
    grad_slots: a tensor (or view) whose element 0 is slot 0's first element; ready: int32 tensor."""
    _check(_lib.smlm_adamw_step_reduce(_ptr(param), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad_slots), int(n_slots),
                                       int(slot_stride), int(own_slot), _ptr(param_bf16), int(n), int(step), lr, beta1,
                                       beta2, eps, weight_decay, grad_scale, max_grad_norm, int(bool(zero_grad)),
                                       _ptr(ready), int(ready_target), _ptr(ws),
                                       0 if ws is None else ws.numel() * ws.element_size(),
                                       _stream(stream, param.device)), "smlm_adamw_step_reduce")


IPC_HANDLE_BYTES = 64


def smlm_ipc_get_handle(t):
    """(CUDA IPC handle (64 bytes) of the allocation holding tensor t, t's byte offset in it)."""
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = ctypes.c_uint64(0)
    _check(_lib.smlm_ipc_get_handle(_ptr(t), buf, ctypes.byref(off)), "smlm_ipc_get_handle")
    return buf.raw, int(off.value)


def smlm_ipc_open_handle(handle: bytes) -> int:
    """Map a peer allocation; returns its base address in this process."""
    out = ctypes.c_void_p(0)
    _check(_lib.smlm_ipc_open_handle(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES), ctypes.byref(out)),
           "smlm_ipc_open_handle")
    return int(out.value)


def smlm_ipc_close_handle(ptr: int):
    _check(_lib.smlm_ipc_close_handle(ptr), "smlm_ipc_close_handle")


def smlm_pool_set_grad_fanout(pool: int, deltas):
    arr = (ctypes.c_int64 * max(len(deltas), 1))(*[int(d) for d in deltas])
    _check(_lib.smlm_pool_set_grad_fanout(pool, len(deltas), ctypes.cast(arr, ctypes.c_void_p)),
           "smlm_pool_set_grad_fanout")


def smlm_fanout_wait(ready, target: int, stream=None):
    _check(_lib.smlm_fanout_wait(_ptr(ready), int(target), _stream(stream, ready.device)), "smlm_fanout_wait")


def smlm_fanout_signal(ready_ptrs, stream=None, device=None):
    """ready_ptrs: device addresses (ints) of every rank's ready counter as mapped in this process."""
    arr = (ctypes.c_void_p * len(ready_ptrs))(*[int(p) for p in ready_ptrs])
    import torch
    st = _stream(stream, device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    _check(_lib.smlm_fanout_signal(len(ready_ptrs), ctypes.cast(arr, ctypes.c_void_p), st), "smlm_fanout_signal")


class AttnBatch:
    """Host segment arrays of an attention call (include/smlm.h smlm_attn_batch), kept alive."""

    def __init__(self, offsets, modes, cache_slots=None, past=None):
        self.offsets = np.ascontiguousarray(offsets, np.int32)
        self.modes = np.ascontiguousarray(modes, np.int8)
        self.cache = None if cache_slots is None else np.ascontiguousarray(cache_slots, np.int32)
        self.past = None if past is None else np.ascontiguousarray(past, np.int32)
        self.c = smlm_attn_batch(int(self.offsets[-1]) if len(self.offsets) else 0, len(self.modes),
                                 self.offsets.ctypes.data, self.modes.ctypes.data,
                                 None if self.cache is None else self.cache.ctypes.data,
                                 None if self.past is None else self.past.ctypes.data)


def smlm_attention_workspace_size(batch: AttnBatch, n_heads: int, n_kv_heads: int) -> int:
    return int(_lib.smlm_attention_workspace_size(ctypes.byref(batch.c), n_heads, n_kv_heads))


def smlm_attention(batch: AttnBatch, Q, K, V, O, K_cache=None, V_cache=None, scale=None, ws=None, stream=None):
    """Q [S, Hq, 128], K/V [S, Hkv, 128], O [S, Hq, 128]; caches [slots, capacity, Hkv, 128] (bf16)."""
    import math
    import torch
    nh, nkv, d = Q.shape[1], K.shape[1], Q.shape[2]
    if ws is None:
        ws = torch.empty(max(smlm_attention_workspace_size(batch, nh, nkv), 256), dtype=torch.uint8, device=Q.device)
    slots = 0 if K_cache is None else K_cache.shape[0]
    cap = 0 if K_cache is None else K_cache.shape[1]
    _check(_lib.smlm_attention(ctypes.byref(batch.c), nh, nkv, d, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(K_cache),
                               _ptr(V_cache), slots, cap, 1.0 / math.sqrt(d) if scale is None else scale, _ptr(ws),
                               ws.numel() * ws.element_size(), _stream(stream, Q.device)), "smlm_attention")


def smlm_launch_count() -> int:
    return int(_lib.smlm_launch_count())


def smlm_profile_enable(mask):
    """Bitmask of kernel classes to time (bool True = all classes)."""
    if isinstance(mask, bool):
        mask = 0x1F if mask else 0
    _lib.smlm_profile_enable(int(mask))


def smlm_profile_read(kind: int):
    ms = ctypes.c_double(0)
    n = ctypes.c_int(0)
    _lib.smlm_profile_read(kind, ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


# ------------------------------ convenience owner ------------------------------
class Pool:
    """One adapter pool per (layer, projection).  Keeps borrowed adapter tensors alive."""

    def __init__(self, in_features: int, out_features: int, rank: int, capacity: int, dtype: int = SMLM_BF16,
                 device: int = 0):
        import torch
        self.device = torch.device("cuda", device)
        self.in_features, self.out_features, self.rank, self.capacity = in_features, out_features, rank, capacity
        self.dtype = dtype
        self.h = smlm_pool_create(device, in_features, out_features, rank, capacity, dtype)
        self._keep = {}
        self._ws = None

    def close(self):
        if self.h:
            smlm_pool_destroy(self.h)
            self.h = None
            self._keep.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register(self, A, B, scale: float, stream=None) -> int:
        """A [r_a, in], B [out, r_a]; r_a below the pool rank registers a lower-rank adapter."""
        if A.shape[0] != self.rank:
            slot = smlm_adapter_register_rank(self.h, A, B, A.shape[0], scale, stream)
        else:
            slot = smlm_adapter_register(self.h, A, B, scale, stream)
        self._keep[slot] = [A, B, None, None]
        return slot

    def set_grad(self, slot: int, dA=None, dB=None):
        smlm_adapter_set_grad(self.h, slot, dA, dB)
        self._keep[slot][2:] = [dA, dB]

    def unregister(self, slot: int, stream=None):
        smlm_adapter_unregister(self.h, slot, stream, self.device)
        self._keep.pop(slot, None)

    def set_option(self, option: int, value: int):
        smlm_pool_set_option(self.h, option, value)

    def workspace(self, batch: Batch, backward: bool = False):
        import torch
        n = smlm_workspace_size(self.h, batch, backward)
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.empty(max(n, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def forward(self, batch: Batch, X, W, Y=None, V_save=None, ws=None, stream=None):
        import torch
        if Y is None:
            Y = torch.empty(X.shape[0], self.out_features, dtype=X.dtype, device=X.device)
        if ws is None:
            ws = self.workspace(batch, False)
        smlm_forward(self.h, batch, X, W, Y, V_save, ws, stream)
        return Y

    def backward(self, batch: Batch, X, W, dY, V_save=None, dX=None, accumulate=False, ws=None, stream=None):
        if ws is None:
            ws = self.workspace(batch, True)
        smlm_backward(self.h, batch, X, W, dY, V_save, dX, accumulate, ws, stream)
        return dX

    def plan(self, batch: Batch, backward: bool = False):
        return smlm_plan_export(self.h, batch, backward)
