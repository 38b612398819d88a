"""Oracle of the Alg. 1 attention branch -- TEST INFRASTRUCTURE ONLY (only
tests/, __graft_entry__.smoke() and bench.py may import it; the product package never does).

PAPER.md P:319-356 (Alg. 1, "Computation flow control in attention layer of Loquetier"): after the
joint Q/K/V projections, the fine-tune rows (F) get the standard attention forward, the prefill and
evaluation rows (P) the FlashInfer prefill forward with "Initialize KVCache for prefills", and the
decode rows (D) "Append KVCache for decodes" and attend over their request's cache.  All three are
the same plain definition -- causal scaled-dot-product attention of a token over the keys of its
own request -- which this module writes out (reading R14):

    for a segment g of mode FINETUNE / EVAL / PREFILL (a fresh sequence, positions 0..L-1):
        o[t, h] = sum_{j <= t} softmax_j(q[t, h] . k[j, kv(h)] * scale) v[j, kv(h)]
        over the segment's own rows j; PREFILL also writes k/v of its rows to cache[c][0..L)
    for a segment g of mode DECODE (request cache c holding n_past tokens):
        row i of the segment is appended at cache position n_past + i, then
        o[t, h] = sum_{j <= n_past + i} softmax_j(q[t, h] . K_c[j, kv(h)] * scale) V_c[j, kv(h)]
    kv(h) = h // (H_q / H_kv)  (grouped-query attention, Llama-3: 32 query heads, 8 KV heads).

Shapes: Q [S, Hq, d], K/V [S, Hkv, d] (row-major, the projections' outputs), O [S, Hq, d];
cache: K_cache / V_cache [n_slots, capacity, Hkv, d].  fp64 arithmetic on the exact input values,
softmax as exp(s - max) / sum in fp64 -- every sum a plain ascending numpy reduction.
"""
from __future__ import annotations

import numpy as np

FINETUNE, EVAL, PREFILL, DECODE = 0, 1, 2, 3


def _f64(t):
    try:
        import torch
        if isinstance(t, torch.Tensor):
            return t.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(t, np.float64)


def _attend(q, k, v, scale):
    """q [Hq, d] one token; k, v [n, Hkv, d] its visible keys -> o [Hq, d]."""
    Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    o = np.zeros((Hq, d))
    for h in range(Hq):
        kh, vh = k[:, h // g, :], v[:, h // g, :]
        s = (kh @ q[h]) * scale
        p = np.exp(s - s.max())
        o[h] = (p / p.sum()) @ vh
    return o


def attention(offsets, modes, cache_slot, n_past, Q, K, V, K_cache, V_cache, scale, rows=None):
    """Returns (O [S, Hq, d] fp64 (rows not computed stay 0 when `rows` is given),
    K_cache', V_cache' (fp64 copies with the prefill rows written and the decode rows appended))."""
    Qd, Kd, Vd = _f64(Q), _f64(K), _f64(V)
    Kc, Vc = _f64(K_cache).copy(), _f64(V_cache).copy()
    S, Hq, d = Qd.shape
    O = np.zeros((S, Hq, d))
    want = None if rows is None else set(int(r) for r in rows)
    G = len(modes)
    # cache writes first (a decode row attends to everything appended before it, itself included)
    for g in range(G):
        a, b = int(offsets[g]), int(offsets[g + 1])
        c = int(cache_slot[g])
        if modes[g] == PREFILL and c >= 0:
            Kc[c, 0:b - a] = Kd[a:b]
            Vc[c, 0:b - a] = Vd[a:b]
        elif modes[g] == DECODE:
            p0 = int(n_past[g])
            Kc[c, p0:p0 + b - a] = Kd[a:b]
            Vc[c, p0:p0 + b - a] = Vd[a:b]
    for g in range(G):
        a, b = int(offsets[g]), int(offsets[g + 1])
        for t in range(a, b):
            if want is not None and t not in want:
                continue
            i = t - a
            if modes[g] == DECODE:
                c, p0 = int(cache_slot[g]), int(n_past[g])
                O[t] = _attend(Qd[t], Kc[c, :p0 + i + 1], Vc[c, :p0 + i + 1], scale)
            else:
                O[t] = _attend(Qd[t], Kd[a:t + 1], Vd[a:t + 1], scale)
    return O, Kc, Vc
