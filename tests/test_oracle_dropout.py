"""Pins of the oracle's LoRA dropout (App. D Table 5 lora_dropout
0.05; reading R13: PEFT's y = W x + s B A dropout(x), dropout on FINETUNE rows only) and
of the counter-based mask generator, against things other than the oracle itself:

  * the hand-worked example with a fixed mask (tests/golden/worked_example_dropout.json)
  * an all-ones mask with p = 0 is the no-dropout oracle, bit for bit
  * rows that are not FINETUNE rows ignore the mask entirely
  * a single fine-tune segment against numpy: Y = X W^T + s ((keep*X/(1-p)) A^T) B^T
  * central finite differences of L = <dY, Y> under the mask (L stays linear in A, B and X, so
    they are exact up to rounding): the backward (dX through the mask, dA from x~, dB from v)
  * the mask generator: drop rate within its binomial bounds, the threshold rule, and
    independence of the mask from the seed's two halves.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import DECODE, EVAL, FINETUNE, PREFILL


@pytest.fixture(scope="module", autouse=True)
def _build():
    oracle.build()


def _rand_case(seed, in_f=11, out_f=9, r=3, U=2, lengths=(4, 3, 5, 2), modes=None, slots=None):
    modes = modes or [FINETUNE, EVAL, FINETUNE, DECODE][:len(lengths)]
    return synth.random_case(seed, in_f, out_f, r, U, list(lengths), modes, slots, dtype=torch.float64)


def test_worked_example_with_mask(golden_dir):
    base = json.load(open(os.path.join(golden_dir, "worked_example.json")))
    d = json.load(open(os.path.join(golden_dir, "worked_example_dropout.json")))
    batch = synth.batch_from_lengths(np.diff(base["offsets"]).tolist(), base["slots"], base["modes"],
                                     base["seg_scale"])
    W = torch.tensor(base["W"], dtype=torch.float64)
    A = [torch.tensor(a, dtype=torch.float64) for a in base["A"]]
    B = [torch.tensor(b, dtype=torch.float64) for b in base["B"]]
    X = torch.tensor(base["X"], dtype=torch.float64)
    dY = torch.tensor(base["dY"], dtype=torch.float64)
    keep = np.array(d["keep"], bool)
    Y, V = oracle.forward(batch, W, A, B, base["slot_scale"], X, keep=keep, p=d["p"])
    assert np.array_equal(Y, np.array(d["expect"]["Y"], np.float64))
    assert np.array_equal(V[0], np.array(d["expect"]["V_ft"]["0"], np.float64))
    dX, dA, dB = oracle.backward(batch, W, A, B, base["slot_scale"], X, dY, keep=keep, p=d["p"])
    assert np.array_equal(dX[0], np.array(d["expect"]["dX_ft"]["0"], np.float64))
    assert np.array_equal(dA, np.array(d["expect"]["dA"], np.float64))
    assert np.array_equal(dB, np.array(d["expect"]["dB"], np.float64))


def test_all_kept_p0_is_no_dropout():
    batch, w, X, dY = _rand_case(1)
    keep = np.ones((batch.S, X.shape[1]), bool)
    Y0, V0 = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    Y1, V1 = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, keep=keep, p=0.0)
    assert np.array_equal(Y0, Y1) and np.array_equal(V0, V1)
    g0 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    g1 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, keep=keep, p=0.0)
    for a, b in zip(g0, g1):
        assert np.array_equal(a, b)


def test_non_finetune_rows_ignore_mask():
    batch, w, X, dY = _rand_case(2, modes=[EVAL, PREFILL, DECODE, FINETUNE], slots=[0, 1, 0, 1])
    keep = synth.dropout_keep(99, 0.5, batch.S, X.shape[1])
    Y0, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    Y1, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, keep=keep, p=0.5)
    ft = batch.ft_rows()
    other = np.setdiff1d(np.arange(batch.S), ft)
    assert np.array_equal(Y0[other], Y1[other])
    assert not np.allclose(Y0[ft], Y1[ft])


@pytest.mark.parametrize("p", [0.05, 0.5])
def test_single_finetune_segment_vs_numpy(p):
    batch, w, X, dY = _rand_case(3, lengths=(7,), modes=[FINETUNE], slots=[1])
    keep = synth.dropout_keep(7, p, batch.S, X.shape[1])
    pe = synth.dropout_effective_p(p)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, keep=keep, p=pe)
    Xn, Wn, An, Bn = X.numpy(), w.W.numpy(), w.A[1].numpy(), w.B[1].numpy()
    Xt = keep * Xn / (1.0 - pe)
    ref = Xn @ Wn.T + w.slot_scale[1] * (Xt @ An.T) @ Bn.T
    assert np.max(np.abs(Y - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.max(np.abs(V - Xt @ An.T)) <= 1e-12 * np.max(np.abs(V))


def _loss(batch, W, A, B, ss, X, dY, keep, p):
    Y, _ = oracle.forward(batch, W, A, B, ss, X, keep=keep, p=p)
    ft = batch.ft_rows()
    return float(np.sum(dY.numpy()[ft] * Y[ft]))


@pytest.mark.parametrize("seed,p", [(4, 0.25), (5, 0.05)])
def test_finite_differences_under_mask(seed, p):
    batch, w, X, dY = _rand_case(seed, lengths=(3, 2, 4, 2), modes=[FINETUNE, DECODE, FINETUNE, EVAL],
                                 slots=[0, 0, 1, 1])
    keep = synth.dropout_keep(1000 + seed, p, batch.S, X.shape[1])
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, keep=keep, p=p)
    h = 0.37
    args = (batch, w.W)
    for a in range(2):
        for (j, k) in [(0, 0), (2, 10), (1, 4)]:
            Ap = [t.clone() for t in w.A]; Am = [t.clone() for t in w.A]
            Ap[a][j, k] += h; Am[a][j, k] -= h
            fd = (_loss(*args, Ap, w.B, w.slot_scale, X, dY, keep, p) -
                  _loss(*args, Am, w.B, w.slot_scale, X, dY, keep, p)) / (2 * h)
            assert abs(fd - dA[a, j, k]) <= 1e-10 * max(1.0, abs(fd))
        for (o, j) in [(0, 0), (8, 2), (3, 1)]:
            Bp = [t.clone() for t in w.B]; Bm = [t.clone() for t in w.B]
            Bp[a][o, j] += h; Bm[a][o, j] -= h
            fd = (_loss(*args, w.A, Bp, w.slot_scale, X, dY, keep, p) -
                  _loss(*args, w.A, Bm, w.slot_scale, X, dY, keep, p)) / (2 * h)
            assert abs(fd - dB[a, o, j]) <= 1e-10 * max(1.0, abs(fd))
    n_dropped = 0
    for t in batch.ft_rows():
        for k in range(X.shape[1]):
            Xp = X.clone(); Xm = X.clone()
            Xp[t, k] += h; Xm[t, k] -= h
            fd = (_loss(*args, w.A, w.B, w.slot_scale, Xp, dY, keep, p) -
                  _loss(*args, w.A, w.B, w.slot_scale, Xm, dY, keep, p)) / (2 * h)
            assert abs(fd - dX[t, k]) <= 1e-10 * max(1.0, abs(fd))
            n_dropped += int(not keep[t, k])
    assert n_dropped > 0   # the check covered dropped elements (their dX is the base term only)


def test_mask_generator_statistics_and_threshold():
    S, n = 257, 4095   # odd widths: pairs never straddle rows (ceil(in/2) pairs per row)
    for p in (0.05, 0.3):
        keep = synth.dropout_keep(0xDEADBEEF12345678, p, S, n)
        drop = 1.0 - keep.mean()
        pe = synth.dropout_effective_p(p)
        sd = np.sqrt(pe * (1 - pe) / keep.size)
        assert abs(drop - pe) <= 6 * sd, (p, drop, pe)
    assert synth.dropout_keep(5, 0.0, 8, 8).all()
    assert synth.dropout_threshold(0.05) == 3277 and synth.dropout_effective_p(0.05) == 3277 / 65536
    # both halves of the 64-bit seed matter; rows and columns are not repeated
    a = synth.dropout_keep(1, 0.5, 16, 64)
    b = synth.dropout_keep(1 + (1 << 32), 0.5, 16, 64)
    c = synth.dropout_keep(2, 0.5, 16, 64)
    assert (a != b).mean() > 0.3 and (a != c).mean() > 0.3
    assert (a[0] != a[1]).mean() > 0.3
    with pytest.raises(ValueError):
        synth.dropout_threshold(1.0)
