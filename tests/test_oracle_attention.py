"""Pins of the attention oracle (oracle/attention.py, Alg. 1)
against things other than itself:
  * torch.nn.functional.scaled_dot_product_attention (causal, library routine) on a prefill
    segment, with the GQA heads expanded -- <= 1e-12
  * a one-token segment returns its own value vector exactly (softmax of one score is 1)
  * zero queries give uniform weights: o[t] = mean of v over the visible keys
  * decode after prefill == the last row of one longer prefill (two code paths: cache vs rows)
  * requests are isolated: a segment's outputs do not depend on the other segments
  * cache writes: a prefill fills rows [0, L) of its slot, a decode appends at n_past
"""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle.attention import DECODE, EVAL, FINETUNE, PREFILL

HQ, HKV, D = 4, 2, 16


def _rand(seed, S, cap=64, slots=3):
    g = torch.Generator().manual_seed(seed)
    Q = torch.randn(S, HQ, D, generator=g, dtype=torch.float64)
    K = torch.randn(S, HKV, D, generator=g, dtype=torch.float64)
    V = torch.randn(S, HKV, D, generator=g, dtype=torch.float64)
    Kc = torch.randn(slots, cap, HKV, D, generator=g, dtype=torch.float64)
    Vc = torch.randn(slots, cap, HKV, D, generator=g, dtype=torch.float64)
    return Q, K, V, Kc, Vc


def test_prefill_vs_torch_sdpa():
    L = 23
    Q, K, V, Kc, Vc = _rand(1, L)
    scale = 1.0 / np.sqrt(D)
    O, _, _ = OA.attention([0, L], [PREFILL], [0], [0], Q, K, V, Kc, Vc, scale)
    rep = HQ // HKV
    q = Q.permute(1, 0, 2)[None]
    k = K.repeat_interleave(rep, dim=1).permute(1, 0, 2)[None]
    v = V.repeat_interleave(rep, dim=1).permute(1, 0, 2)[None]
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=scale)[0].permute(1, 0, 2)
    assert np.max(np.abs(O - ref.numpy())) <= 1e-12 * np.max(np.abs(ref.numpy()))


def test_single_token_and_uniform_weights():
    Q, K, V, Kc, Vc = _rand(2, 9)
    O, _, _ = OA.attention([0, 1, 9], [EVAL, FINETUNE], [-1, -1], [0, 0], Q, K, V, Kc, Vc, 0.3)
    rep = HQ // HKV
    for h in range(HQ):
        assert np.array_equal(O[0, h], V[0, h // rep].numpy())
    Qz = torch.zeros_like(Q)
    O2, _, _ = OA.attention([0, 9], [FINETUNE], [-1], [0], Qz, K, V, Kc, Vc, 0.3)
    for t in range(9):
        for h in range(HQ):
            assert np.allclose(O2[t, h], V[:t + 1, h // rep].numpy().mean(0), rtol=0, atol=1e-14)


def test_decode_after_prefill_equals_longer_prefill():
    L = 17
    Q, K, V, Kc, Vc = _rand(3, L + 1)
    scale = 0.25
    # one prefill of L + 1 tokens
    O_full, _, _ = OA.attention([0, L + 1], [PREFILL], [1], [0], Q, K, V, Kc, Vc, scale)
    # prefill of L tokens into slot 1, then one decode token appended at position L
    _, Kc1, Vc1 = OA.attention([0, L], [PREFILL], [1], [0], Q[:L], K[:L], V[:L], Kc, Vc, scale)
    O_dec, Kc2, Vc2 = OA.attention([0, 1], [DECODE], [1], [L], Q[L:], K[L:], V[L:], Kc1, Vc1, scale)
    assert np.max(np.abs(O_dec[0] - O_full[L])) <= 1e-13
    assert np.array_equal(Kc2[1, :L + 1], K.numpy()) and np.array_equal(Vc2[1, :L + 1], V.numpy())
    # untouched: other slots and positions past the appended token
    assert np.array_equal(Kc2[0], Kc.numpy()[0]) and np.array_equal(Kc2[1, L + 1:], Kc.numpy()[1, L + 1:])


def test_segments_are_isolated():
    Q, K, V, Kc, Vc = _rand(4, 30)
    offs, modes, slots, past = [0, 10, 13, 30], [FINETUNE, DECODE, PREFILL], [-1, 0, 2], [0, 7, 0]
    O, _, _ = OA.attention(offs, modes, slots, past, Q, K, V, Kc, Vc, 0.2)
    for g in range(3):
        a, b = offs[g], offs[g + 1]
        Og, _, _ = OA.attention([0, b - a], [modes[g]], [slots[g]], [past[g]], Q[a:b], K[a:b], V[a:b], Kc, Vc, 0.2)
        assert np.array_equal(Og, O[a:b])
    # a decode segment of several tokens attends causally to the cache plus its earlier tokens
    O3, Kc3, _ = OA.attention([0, 3], [DECODE], [0], [5], Q[:3], K[:3], V[:3], Kc, Vc, 0.2)
    assert np.array_equal(Kc3[0, 5:8], K[:3].numpy())
    O4, _, _ = OA.attention([0, 1], [DECODE], [0], [7], Q[2:3], K[2:3], V[2:3], Kc3, Vc, 0.2)
    Vc3 = Vc.clone().numpy()
    Vc3[0, 5:8] = V[:3].numpy()
    O5, _, _ = OA.attention([0, 1], [DECODE], [0], [7], Q[2:3], K[2:3], V[2:3], Kc3, Vc3, 0.2)
    assert np.max(np.abs(O5[0] - O3[2])) <= 1e-13
