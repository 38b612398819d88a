"""GPU parity of the Alg. 1 attention branch against the fp64
oracle (oracle/attention.py): a packed batch of FINETUNE / EVAL / PREFILL segments (causal, the
tcgen05 kernel; one PREFILL initialises its KV cache) and DECODE segments (append + attend over the
cache), Llama-3 grouped-query heads, bf16 tolerance 2e-2 (tests/util.py), cache writes bit-exact."""
import math

import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle.attention import DECODE, EVAL, FINETUNE, PREFILL
from tests.util import BF16_TOL, parity_err

pytestmark = pytest.mark.gpu


def _case(seed, lengths, modes, slots, past, hq=8, hkv=2, cap=512, n_slots=4):
    g = torch.Generator().manual_seed(seed)
    S = sum(lengths)
    Q = torch.randn(S, hq, 128, generator=g).to(torch.bfloat16)
    K = torch.randn(S, hkv, 128, generator=g).to(torch.bfloat16)
    V = torch.randn(S, hkv, 128, generator=g).to(torch.bfloat16)
    Kc = torch.randn(n_slots, cap, hkv, 128, generator=g).to(torch.bfloat16)
    Vc = torch.randn(n_slots, cap, hkv, 128, generator=g).to(torch.bfloat16)
    offs = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
    return offs, Q, K, V, Kc, Vc


def _run(offs, modes, slots, past, Q, K, V, Kc, Vc):
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    b = S.AttnBatch(offs, modes, slots, past)
    O = torch.full(Q.shape, float("nan"), dtype=torch.bfloat16, device=dev)
    Kd, Vd = Kc.to(dev), Vc.to(dev)
    S.smlm_attention(b, Q.to(dev), K.to(dev), V.to(dev), O, Kd, Vd)
    torch.cuda.synchronize()
    return O.cpu(), Kd.cpu(), Vd.cpu()


@pytest.mark.parametrize("hq,hkv", [(8, 2), (4, 4), (32, 8), (8, 4), (16, 2)])
def test_mixed_batch_attention(hq, hkv):
    lengths = [200, 70, 300, 1, 3, 129, 1]
    modes = [FINETUNE, EVAL, PREFILL, DECODE, DECODE, PREFILL, DECODE]
    slots = [-1, -1, 0, 1, 2, -1, 3]
    past = [0, 0, 0, 150, 40, 0, 511]
    offs, Q, K, V, Kc, Vc = _case(7 + hq, lengths, modes, slots, past, hq, hkv)
    O, Kd, Vd = _run(offs, modes, slots, past, Q, K, V, Kc, Vc)
    Or, Kr, Vr = OA.attention(offs, modes, slots, past, Q, K, V, Kc, Vc, 1.0 / math.sqrt(128))
    assert not torch.isnan(O).any()
    for g in range(len(modes)):
        a, bnd = offs[g], offs[g + 1]
        assert parity_err(O[a:bnd], Or[a:bnd]) <= BF16_TOL, (g, parity_err(O[a:bnd], Or[a:bnd]))
    # the cache writes are copies: bit-exact, and nothing else in the caches moved
    assert np.array_equal(Kd.double().numpy(), Kr) and np.array_equal(Vd.double().numpy(), Vr)


@pytest.mark.parametrize("hq,hkv", [(8, 2), (4, 4), (16, 2)])
def test_multi_row_decode_segments(hq, hkv):
    """DECODE segments of many rows (several row groups per segment: kAttnDecCols / G rows share one
    read of the slot's K / V) whose rows straddle 128-key chunk boundaries: row i of a segment sees
    cache[0 .. past + i], so rows of one group see different key counts in the boundary chunk."""
    lengths = [37, 5, 70, 9]
    modes = [DECODE, DECODE, DECODE, DECODE]
    slots = [0, 1, 2, 3]
    past = [120, 0, 250, 380]
    offs, Q, K, V, Kc, Vc = _case(17 + hq, lengths, modes, slots, past, hq, hkv)
    O, Kd, Vd = _run(offs, modes, slots, past, Q, K, V, Kc, Vc)
    Or, Kr, Vr = OA.attention(offs, modes, slots, past, Q, K, V, Kc, Vc, 1.0 / math.sqrt(128))
    assert not torch.isnan(O).any()
    for g in range(len(modes)):
        a, bnd = offs[g], offs[g + 1]
        assert parity_err(O[a:bnd], Or[a:bnd]) <= BF16_TOL, (g, parity_err(O[a:bnd], Or[a:bnd]))
    assert np.array_equal(Kd.double().numpy(), Kr) and np.array_equal(Vd.double().numpy(), Vr)


@pytest.mark.parametrize("hq,hkv", [(32, 8), (8, 2)])
def test_decode_chunk_aligned_and_capacity_edge(hq, hkv):
    """DECODE segments whose new rows start exactly at a 128-key chunk boundary (that chunk holds
    no cached row: the kernel skips its cache load and takes every visible row from K / V), span
    two chunks, or end at the last cache position; the caches must equal the oracle's bit for bit
    (the appended rows written once per KV head, nothing else touched)."""
    lengths = [9, 40, 12, 1, 3]
    modes = [DECODE] * 5
    slots = [0, 1, 2, 3, 4]
    past = [256, 100, 500, 384, 0]   # chunk-aligned, straddling 128, up to cap - 1, aligned single, empty cache
    offs, Q, K, V, Kc, Vc = _case(29 + hq, lengths, modes, slots, past, hq, hkv, cap=512, n_slots=5)
    O, Kd, Vd = _run(offs, modes, slots, past, Q, K, V, Kc, Vc)
    Or, Kr, Vr = OA.attention(offs, modes, slots, past, Q, K, V, Kc, Vc, 1.0 / math.sqrt(128))
    assert not torch.isnan(O).any()
    for g in range(len(modes)):
        a, bnd = offs[g], offs[g + 1]
        assert parity_err(O[a:bnd], Or[a:bnd]) <= BF16_TOL, (g, parity_err(O[a:bnd], Or[a:bnd]))
    assert np.array_equal(Kd.double().numpy(), Kr) and np.array_equal(Vd.double().numpy(), Vr)


def test_long_prefill_many_blocks_and_empty_segments():
    lengths = [0, 777, 0, 5]
    modes = [PREFILL, FINETUNE, DECODE, EVAL]
    slots = [0, -1, 1, -1]
    past = [0, 0, 10, 0]
    offs, Q, K, V, Kc, Vc = _case(11, lengths, modes, slots, past)
    O, _, _ = _run(offs, modes, slots, past, Q, K, V, Kc, Vc)
    rows = np.unique(np.concatenate([np.arange(0, 782, 37), [0, 127, 128, 255, 256, 776, 777, 781]]))
    Or, _, _ = OA.attention(offs, modes, slots, past, Q, K, V, Kc, Vc, 1.0 / math.sqrt(128), rows=rows)
    assert parity_err(O[rows], Or[rows]) <= BF16_TOL


def test_decode_matches_prefill_of_the_whole_sequence():
    """A prefill that fills the cache, then a decode token over it, equals row L of one prefill of
    L + 1 tokens computed by the tcgen05 prefill kernel (two kernels, one definition)."""
    from paper_2511_00101_b200 import smlm as S
    L = 300
    offs, Q, K, V, Kc, Vc = _case(13, [L + 1], [PREFILL], [0], [0])
    O_full, _, _ = _run(offs, [PREFILL], [0], [0], Q, K, V, Kc, Vc)
    _, Kd, Vd = _run(np.array([0, L], np.int32), [PREFILL], [0], [0], Q[:L], K[:L], V[:L], Kc, Vc)
    O_dec, _, _ = _run(np.array([0, 1], np.int32), [DECODE], [0], [L], Q[L:], K[L:], V[L:], Kd, Vd)
    assert parity_err(O_dec[0], O_full[L]) <= BF16_TOL


def test_attention_errors():
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    Q = torch.zeros(4, 8, 128, dtype=torch.bfloat16, device=dev)
    K = torch.zeros(4, 3, 128, dtype=torch.bfloat16, device=dev)
    with pytest.raises(S.SmlmError):   # 8 heads over 3 KV heads
        S.smlm_attention(S.AttnBatch([0, 4], [PREFILL]), Q, K, K, Q.clone())
    K2 = torch.zeros(4, 2, 128, dtype=torch.bfloat16, device=dev)
    with pytest.raises(S.SmlmError):   # a decode row without a cache
        S.smlm_attention(S.AttnBatch([0, 4], [DECODE], [0], [0]), Q, K2, K2, Q.clone())
