"""Pins of the fp64 oracle against things other than itself (SURVEY.md §8(c) "What pins each part").

Each pin is chosen so that a plausible mistake (dropped term, wrong sign, wrong index, transposed
operand, wrong scale composition, wrong mode mask) fails at least one of them:
  * hand-worked example (tests/golden/worked_example.json)        -> every term and sign
  * B = 0 equals numpy X W^T                                        -> base term, layout of W
  * single segment/adapter equals numpy X (W + s B A)^T             -> LoRA term, A/B orientation
  * finite differences of L = <dY, Y> (linear in A, B, X: exact)   -> backward vs forward
  * special cases: dY = 0, empty grad mask, seg_scale vs slot_scale -> masking, scale composition
  * permutation invariance, linearity over segments                 -> segment bookkeeping
  * Euler / bilinearity identities at moderate size                 -> gradient consistency
  * C1 checksums computed independently in the survey session       -> recipe + everything
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import DECODE, EVAL, FINETUNE, PREFILL


def _wx(path):
    with open(path) as f:
        return json.load(f)


def _case_from_json(d):
    batch = synth.batch_from_lengths(np.diff(d["offsets"]).tolist(), d["slots"], d["modes"], d["seg_scale"])
    W = torch.tensor(d["W"], dtype=torch.float64)
    A = [torch.tensor(a, dtype=torch.float64) for a in d["A"]]
    B = [torch.tensor(b, dtype=torch.float64) for b in d["B"]]
    X = torch.tensor(d["X"], dtype=torch.float64)
    dY = torch.tensor(d["dY"], dtype=torch.float64)
    return batch, W, A, B, d["slot_scale"], X, dY


def test_worked_example(golden_dir):
    d = _wx(os.path.join(golden_dir, "worked_example.json"))
    batch, W, A, B, ss, X, dY = _case_from_json(d)
    Y, V = oracle.forward(batch, W, A, B, ss, X)
    assert np.array_equal(Y, np.array(d["expect"]["Y"], float))
    for row, v in d["expect"]["V_ft"].items():
        assert np.array_equal(V[int(row)], np.array(v, float))
    # V_save only for fine-tune rows
    assert np.all(V[1:] == 0)
    dX, dA, dB = oracle.backward(batch, W, A, B, ss, X, dY)
    for row, v in d["expect"]["dX_ft"].items():
        assert np.array_equal(dX[int(row)], np.array(v, float))
    assert np.all(dX[1:] == 0)  # non fine-tune rows untouched
    assert np.array_equal(dA, np.array(d["expect"]["dA"], float))
    assert np.array_equal(dB, np.array(d["expect"]["dB"], float))


def _rand_case(seed, in_f=24, out_f=20, r=4, U=3, lengths=(5, 7, 3, 6), modes=None, slots=None,
               seg_scale=None):
    modes = modes or [FINETUNE, EVAL, FINETUNE, DECODE][:len(lengths)]
    return synth.random_case(seed, in_f, out_f, r, U, list(lengths), modes, slots, seg_scale,
                             dtype=torch.float64)


def test_b_zero_equals_base_matmul():
    batch, w, X, dY = _rand_case(1, slots=[0, 1, 2, 0])
    Bz = [torch.zeros_like(b) for b in w.B]
    Y, _ = oracle.forward(batch, w.W, w.A, Bz, w.slot_scale, X)
    ref = X.numpy() @ w.W.numpy().T
    assert np.max(np.abs(Y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("mode", [FINETUNE, EVAL, PREFILL, DECODE])
def test_single_segment_dense(mode):
    g = torch.Generator().manual_seed(7)
    in_f, out_f, r, S = 33, 17, 5, 11
    W = torch.randn(out_f, in_f, generator=g, dtype=torch.float64)
    A = torch.randn(r, in_f, generator=g, dtype=torch.float64)
    B = torch.randn(out_f, r, generator=g, dtype=torch.float64)
    X = torch.randn(S, in_f, generator=g, dtype=torch.float64)
    s = 1.75
    batch = synth.batch_from_lengths([S], [0], [mode])
    Y, _ = oracle.forward(batch, W, [A], [B], [s], X)
    ref = X.numpy() @ (W.numpy() + s * B.numpy() @ A.numpy()).T
    assert np.max(np.abs(Y - ref)) <= 1e-12 * np.max(np.abs(ref))
    # two-step low rank identity (SPEC-style invariant): (X A^T) B^T == X (B A)^T
    two = X.numpy() @ A.numpy().T @ B.numpy().T
    assert np.allclose(two, X.numpy() @ (B.numpy() @ A.numpy()).T, rtol=0, atol=1e-10)


def test_inplace_base_mode():
    batch, w, X, dY = _rand_case(2, slots=[2, 0, -1, 1])
    Y1, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    base = torch.from_numpy(X.numpy() @ w.W.numpy().T)
    Y2, _ = oracle.forward(batch, None, w.A, w.B, w.slot_scale, X, Y_in=base)
    assert np.max(np.abs(Y1 - Y2)) <= 1e-12 * np.max(np.abs(Y1))


def _loss(batch, W, A, B, ss, X, dY):
    Y, _ = oracle.forward(batch, W, A, B, ss, X)
    # loss only sees fine-tune rows: other rows carry no gradient
    ft = batch.ft_rows()
    return float(np.sum(dY.numpy()[ft] * Y[ft]))


@pytest.mark.parametrize("seed", [3, 4])
def test_finite_differences(seed):
    """L = <dY, Y> over fine-tune rows is linear in each of A, B, X: central differences are exact
    up to rounding for any step (h = 0.37)."""
    batch, w, X, dY = _rand_case(seed, in_f=9, out_f=7, r=3, U=2, lengths=(3, 2, 4, 2),
                                 modes=[FINETUNE, DECODE, FINETUNE, EVAL], slots=[0, 0, 1, 1],
                                 seg_scale=[1.0, 2.0, 0.5, 1.0])
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    h = 0.37
    for a in range(2):
        for (j, k) in [(0, 0), (2, 8), (1, 4)]:
            Ap = [t.clone() for t in w.A]; Am = [t.clone() for t in w.A]
            Ap[a][j, k] += h; Am[a][j, k] -= h
            fd = (_loss(batch, w.W, Ap, w.B, w.slot_scale, X, dY) -
                  _loss(batch, w.W, Am, w.B, w.slot_scale, X, dY)) / (2 * h)
            assert abs(fd - dA[a, j, k]) <= 1e-10 * max(1.0, abs(fd))
        for (o, j) in [(0, 0), (6, 2), (3, 1)]:
            Bp = [t.clone() for t in w.B]; Bm = [t.clone() for t in w.B]
            Bp[a][o, j] += h; Bm[a][o, j] -= h
            fd = (_loss(batch, w.W, w.A, Bp, w.slot_scale, X, dY) -
                  _loss(batch, w.W, w.A, Bm, w.slot_scale, X, dY)) / (2 * h)
            assert abs(fd - dB[a, o, j]) <= 1e-10 * max(1.0, abs(fd))
    for t in batch.ft_rows():
        for k in [0, 5, 8]:
            Xp = X.clone(); Xm = X.clone()
            Xp[t, k] += h; Xm[t, k] -= h
            fd = (_loss(batch, w.W, w.A, w.B, w.slot_scale, Xp, dY) -
                  _loss(batch, w.W, w.A, w.B, w.slot_scale, Xm, dY)) / (2 * h)
            assert abs(fd - dX[t, k]) <= 1e-10 * max(1.0, abs(fd))


def test_dy_zero_and_masking():
    batch, w, X, dY = _rand_case(5, slots=[0, 1, 2, 0], modes=[FINETUNE, FINETUNE, FINETUNE, DECODE])
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, torch.zeros_like(dY))
    assert np.all(dX == 0) and np.all(dA == 0) and np.all(dB == 0)
    # empty grad mask: dA/dB untouched (stay exactly zero), dX still the full gradient
    dX1, dA1, dB1 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, has_grad=[0, 0, 0])
    dX2, _, _ = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    assert np.all(dA1 == 0) and np.all(dB1 == 0)
    assert np.array_equal(dX1, dX2)
    # partial mask: masked slot untouched, others equal the unmasked result
    _, dA3, dB3 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, has_grad=[1, 0, 1])
    _, dA4, dB4 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    assert np.all(dA3[1] == 0) and np.array_equal(dA3[0], dA4[0]) and np.array_equal(dB3[2], dB4[2])


def test_untouched_slot_and_accumulate():
    batch, w, X, dY = _rand_case(6, slots=[0, 0, 1, 1], modes=[FINETUNE, EVAL, FINETUNE, DECODE])
    pre_dA = np.full((3, 4, 24), 7.0)
    pre_dB = np.full((3, 20, 4), -3.0)
    _, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, dA_in=pre_dA, dB_in=pre_dB)
    assert np.all(dA[2] == 7.0) and np.all(dB[2] == -3.0)  # slot 2 has no fine-tune rows
    _, dA0, dB0 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    _, dAacc, _ = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, dA_in=pre_dA,
                                  dB_in=pre_dB, accumulate=True)
    assert np.allclose(dAacc[:2], dA0[:2] + 7.0, rtol=0, atol=1e-12)


def test_seg_scale_equals_halved_slot_scale():
    batch, w, X, dY = _rand_case(8, slots=[0, 1, 0, 1], seg_scale=[0.5, 0.5, 0.5, 0.5])
    Y1, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    _, dA1, dB1 = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    b2 = synth.Batch(batch.offsets, batch.slots, batch.modes, None)
    half = [s * 0.5 for s in w.slot_scale]
    Y2, _ = oracle.forward(b2, w.W, w.A, w.B, half, X)
    _, dA2, dB2 = oracle.backward(b2, w.W, w.A, w.B, half, X, dY)
    assert np.array_equal(Y1, Y2) and np.array_equal(dA1, dA2) and np.array_equal(dB1, dB2)


def test_permutation_invariance():
    lengths = [5, 7, 3, 6, 4]
    slots = [0, 1, 2, 0, -1]
    modes = [FINETUNE, EVAL, FINETUNE, DECODE, FINETUNE]
    batch, w, X, dY = _rand_case(9, lengths=lengths, slots=slots, modes=modes)
    Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    perm = [3, 0, 4, 2, 1]
    rows = np.concatenate([np.arange(batch.offsets[g], batch.offsets[g + 1]) for g in perm])
    pb = synth.batch_from_lengths([lengths[g] for g in perm], [slots[g] for g in perm],
                                  [modes[g] for g in perm])
    Yp, _ = oracle.forward(pb, w.W, w.A, w.B, w.slot_scale, X[rows])
    dXp, dAp, dBp = oracle.backward(pb, w.W, w.A, w.B, w.slot_scale, X[rows], dY[rows])
    assert np.array_equal(Yp, Y[rows])       # per-row arithmetic: bit-exact
    assert np.array_equal(dXp, dX[rows])
    assert np.allclose(dAp, dA, rtol=1e-12, atol=1e-12)  # summation order over tokens changes
    assert np.allclose(dBp, dB, rtol=1e-12, atol=1e-12)


def test_linearity_over_segments():
    batch, w, X, dY = _rand_case(10, lengths=(6, 5), slots=[1, 1], modes=[FINETUNE, FINETUNE])
    _, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    parts = []
    for g in range(2):
        a, b = batch.offsets[g], batch.offsets[g + 1]
        bg = synth.batch_from_lengths([b - a], [1], [FINETUNE])
        parts.append(oracle.backward(bg, w.W, w.A, w.B, w.slot_scale, X[a:b], dY[a:b]))
    assert np.allclose(dA[1], parts[0][1][1] + parts[1][1][1], rtol=1e-12, atol=1e-12)
    assert np.allclose(dB[1], parts[0][2][1] + parts[1][2][1], rtol=1e-12, atol=1e-12)


def test_euler_identities():
    """Y is linear in X, in A alone and in B alone: <dA_a,A_a> = <dB_a,B_a> = <dY, dY_lora_a>
    over a's fine-tune rows, and <dX, X> = <dY, Y> over all fine-tune rows."""
    lengths = [40, 13, 30, 9, 22]
    slots = [0, 0, 1, 0, -1]
    modes = [FINETUNE, DECODE, FINETUNE, FINETUNE, FINETUNE]
    batch, w, X, dY = synth.random_case(11, 96, 80, 8, 2, lengths, modes, slots, dtype=torch.float64)
    Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    base = X.numpy() @ w.W.numpy().T
    rs = batch.row_slot()
    rm = batch.row_mode()
    for a in range(2):
        m = (rs == a) & (rm == FINETUNE)
        rhs = float(np.sum(dY.numpy()[m] * (Y - base)[m]))
        assert abs(np.sum(dA[a] * w.A[a].numpy()) - rhs) <= 1e-10 * max(1, abs(rhs))
        assert abs(np.sum(dB[a] * w.B[a].numpy()) - rhs) <= 1e-10 * max(1, abs(rhs))
    ft = rm == FINETUNE
    lhs = float(np.sum(dX[ft] * X.numpy()[ft]))
    rhs = float(np.sum(dY.numpy()[ft] * Y[ft]))
    assert abs(lhs - rhs) <= 1e-10 * max(1, abs(rhs))


def test_c1_checksums(golden_dir):
    ref = _wx(os.path.join(golden_dir, "c1_checksums.json"))
    batch, w, X, dY = synth.c1_inputs()
    assert np.allclose(X[0, :4].double().numpy(), ref["X0_first4"], rtol=1e-9)
    assert abs(float(w.W[0, 0]) - ref["W00"]) <= 1e-9
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    ft = batch.ft_rows()

    def close(v, r):
        return abs(v - r) <= 1e-10 * abs(r)
    assert close(Y.sum(), ref["sum_Y"]) and close(np.abs(Y).sum(), ref["sum_abs_Y"])
    assert np.allclose(Y[0, :3], ref["Y0_first3"], rtol=1e-10)
    assert np.allclose(Y[31, :3], ref["Y31_first3"], rtol=1e-10)
    assert close(V[ft].sum(), ref["sum_V_ft"])
    assert close(dX[ft].sum(), ref["sum_dX_ft"]) and close(np.abs(dX[ft]).sum(), ref["sum_abs_dX_ft"])
    assert close(dA[0].sum(), ref["sum_dA0"]) and close(np.abs(dA[0]).sum(), ref["sum_abs_dA0"])
    assert close(dB[0].sum(), ref["sum_dB0"]) and close(np.abs(dB[0]).sum(), ref["sum_abs_dB0"])
    assert np.all(dA[1:] == 0) and np.all(dB[1:] == 0)
    assert close(float(np.sum(dA[0] * w.A[0].double().numpy())), ref["euler_a0"])
    assert close(float(np.sum(dB[0] * w.B[0].double().numpy())), ref["euler_a0"])


def test_row_sampling_matches_full():
    batch, w, X, dY = _rand_case(12, lengths=(9, 4, 11), slots=[0, 1, 2], modes=[FINETUNE, DECODE, FINETUNE])
    rows = synth.sample_rows(batch, every=5)
    Yf, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    Ys, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, rows=rows)
    assert np.array_equal(Ys[rows], Yf[rows])
    dXf, _, _ = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY)
    dXs, _, _ = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, rows=rows)
    assert np.array_equal(dXs[rows], dXf[rows])


def test_heterogeneous_ranks_brute_force():
    """SURVEY §8 f2 (heterogeneous ranks in one layer): the zero-padded oracle equals a
    per-row numpy evaluation with each adapter's own rank, and the padded gradient entries are 0."""
    rng = np.random.default_rng(3)
    in_f, out_f, ranks = 12, 10, [4, 8, 2]
    W = rng.standard_normal((out_f, in_f))
    A = [rng.standard_normal((r, in_f)) for r in ranks]
    B = [rng.standard_normal((out_f, r)) for r in ranks]
    ss = [0.5, 2.0, -1.5]
    lengths, slots, modes = [3, 2, 4, 1, 2], [0, 1, 2, -1, 1], [FINETUNE, DECODE, FINETUNE, PREFILL, FINETUNE]
    batch = synth.batch_from_lengths(lengths, slots, modes, [1.0, 1.0, 0.5, 1.0, 2.0])
    X = rng.standard_normal((batch.S, in_f))
    dY = rng.standard_normal((batch.S, out_f))
    Y, _ = oracle.forward(batch, torch.tensor(W), [torch.tensor(a) for a in A], [torch.tensor(b) for b in B], ss,
                          torch.tensor(X))
    dX, dA, dB = oracle.backward(batch, torch.tensor(W), [torch.tensor(a) for a in A], [torch.tensor(b) for b in B],
                                 ss, torch.tensor(X), torch.tensor(dY))
    Yb = X @ W.T
    dXb = np.zeros_like(X)
    dAb = [np.zeros_like(a) for a in A]
    dBb = [np.zeros_like(b) for b in B]
    for g in range(batch.G):
        a = slots[g]
        for t in range(batch.offsets[g], batch.offsets[g + 1]):
            if a >= 0:
                s = ss[a] * batch.seg_scale[g]
                Yb[t] += s * B[a] @ (A[a] @ X[t])
            if modes[g] == FINETUNE:
                dXb[t] = W.T @ dY[t]
                if a >= 0:
                    u = B[a].T @ dY[t]
                    dXb[t] += s * A[a].T @ u
                    dAb[a] += s * np.outer(u, X[t])
                    dBb[a] += s * np.outer(dY[t], A[a] @ X[t])
    np.testing.assert_allclose(Y, Yb, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dX, dXb, rtol=1e-12, atol=1e-12)
    for a, r in enumerate(ranks):
        np.testing.assert_allclose(dA[a, :r], dAb[a], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(dB[a, :, :r], dBb[a], rtol=1e-12, atol=1e-12)
        assert np.all(dA[a, r:] == 0) and np.all(dB[a, :, r:] == 0)
