"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded inputs.

Bar (BASELINE.json north_star): plan/index bookkeeping bit-exact; floating outputs within 2e-2
(bf16 inputs, fp32 accumulate) and 1e-5 (fp32 test mode) under the rms-floored relative metric
of tests/util.parity_err (reading R4).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import plan as plan_oracle
from synth import DECODE, EVAL, FINETUNE, PREFILL
from tests.smlm_run import run_smlm
from tests.util import BF16_TOL, FP32_TOL, parity_err

pytestmark = pytest.mark.gpu


def _oracle_all(batch, w, X, dY, rows=None, has_grad=None, base_in=None, w_null=False):
    Y, V = oracle.forward(batch, None if w_null else w.W, w.A, w.B, w.slot_scale, X, rows=rows, Y_in=base_in)
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, has_grad=has_grad, rows=rows)
    return Y, V, dX, dA, dB


def _check(res, batch, w, X, dY, tol, rows=None, has_grad=None, check_v=True, base_in=None, w_null=False):
    Y, V, dX, dA, dB = _oracle_all(batch, w, X, dY, rows, has_grad, base_in, w_null)
    sel = np.arange(batch.S) if rows is None else np.asarray(rows)
    errs = {"Y": parity_err(res.Y.double().numpy()[sel], Y[sel])}
    ft = batch.ft_rows()
    ftsel = np.intersect1d(ft, sel)
    rs = batch.row_slot()
    ft_lora = ftsel[rs[ftsel] >= 0]
    if check_v and res.V is not None and len(ft_lora):
        errs["V"] = parity_err(res.V.double().numpy()[ft_lora], V[ft_lora])
    if res.dX is not None and len(ftsel):
        errs["dX"] = parity_err(res.dX.double().numpy()[ftsel], dX[ftsel])
    for a in range(len(w.A)):
        if np.any(rs[ft] == a) and (has_grad is None or has_grad[a]):
            errs[f"dA{a}"] = parity_err(res.dA[a].double().numpy(), dA[a])
            errs[f"dB{a}"] = parity_err(res.dB[a].double().numpy(), dB[a])
        else:
            assert torch.all(res.dA[a] == 0) and torch.all(res.dB[a] == 0), f"slot {a} must stay untouched"
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"parity failures {bad} (all: {errs})"
    return errs


# ------------------------------------------------------------------------------------------
# fp32 test mode (1e-5)
# ------------------------------------------------------------------------------------------
def test_c1_fp32(golden_dir):
    batch, w, X, dY = synth.c1_inputs()
    res = run_smlm(batch, w, X, dY)
    _check(res, batch, w, X, dY, FP32_TOL)
    ref = json.load(open(os.path.join(golden_dir, "c1_checksums.json")))
    ft = batch.ft_rows()
    assert abs(res.Y.double().sum().item() - ref["sum_Y"]) <= 1e-4 * abs(ref["sum_Y"]) + 1e-3
    assert abs(res.dA[0].double().sum().item() - ref["sum_dA0"]) <= 1e-4 * abs(ref["sum_dA0"])
    assert abs(res.dX[ft].double().sum().item() - ref["sum_dX_ft"]) <= 1e-4 * abs(ref["sum_dX_ft"])
    assert torch.all(res.dA[1:] == 0) and torch.all(res.dB[1:] == 0)


def _worked(golden_dir, dtype, pad_in=None, pad_out=None, pad_r=None):
    d = json.load(open(os.path.join(golden_dir, "worked_example.json")))
    in_f, out_f, r = d["in"], d["out"], d["rank"]
    pin, pout, pr = pad_in or in_f, pad_out or out_f, pad_r or r
    W = torch.zeros(pout, pin); W[:out_f, :in_f] = torch.tensor(d["W"], dtype=torch.float32)
    A = [torch.zeros(pr, pin) for _ in d["A"]]
    B = [torch.zeros(pout, pr) for _ in d["B"]]
    for i in range(len(A)):
        A[i][:r, :in_f] = torch.tensor(d["A"][i], dtype=torch.float32)
        B[i][:out_f, :r] = torch.tensor(d["B"][i], dtype=torch.float32)
    X = torch.zeros(4, pin); X[:, :in_f] = torch.tensor(d["X"], dtype=torch.float32)
    dY = torch.zeros(4, pout); dY[:, :out_f] = torch.tensor(d["dY"], dtype=torch.float32)
    w = synth.Weights(W.to(dtype), [a.to(dtype) for a in A], [b.to(dtype) for b in B], d["slot_scale"])
    batch = synth.batch_from_lengths(np.diff(d["offsets"]).tolist(), d["slots"], d["modes"], d["seg_scale"])
    return d, batch, w, X.to(dtype), dY.to(dtype), in_f, out_f, r


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_worked_example_exact(golden_dir, dtype):
    pads = (None, None, None) if dtype == torch.float32 else (64, 64, 8)
    d, batch, w, X, dY, in_f, out_f, r = _worked(golden_dir, dtype, *pads)
    res = run_smlm(batch, w, X, dY)
    e = d["expect"]
    assert torch.equal(res.Y[:, :out_f].float(), torch.tensor(e["Y"], dtype=torch.float32))
    assert torch.all(res.Y[:, out_f:] == 0)
    assert torch.equal(res.V[0, :r].float(), torch.tensor(e["V_ft"]["0"], dtype=torch.float32))
    assert torch.equal(res.dX[0, :in_f].float(), torch.tensor(e["dX_ft"]["0"], dtype=torch.float32))
    assert torch.all(res.dX[1:] == 0)  # non fine-tune rows untouched
    assert torch.equal(res.dA[:, :r, :in_f], torch.tensor(e["dA"], dtype=torch.float32))
    assert torch.equal(res.dB[:, :out_f, :r], torch.tensor(e["dB"], dtype=torch.float32))


# ------------------------------------------------------------------------------------------
# bf16 tensor-core path at sizes the oracle finishes quickly (several tiles + ragged tails)
# ------------------------------------------------------------------------------------------
MIXED_LENGTHS = [300, 5, 1, 1, 64, 2, 130, 0, 63, 1, 200, 3, 1]
MIXED_MODES = [FINETUNE, DECODE, DECODE, DECODE, EVAL, DECODE, FINETUNE, DECODE, PREFILL, DECODE, PREFILL,
               FINETUNE, DECODE]


@pytest.mark.parametrize("r", [8, 16, 32, 64])
@pytest.mark.parametrize("shape", [(256, 320), (512, 192)])
def test_bf16_mixed(r, shape):
    in_f, out_f = shape
    slots = [0, 1, 2, 1, 3, -1, 2, 0, 3, 4, -1, 4, 0]
    scale = [1.0, 0.5, 1.0, 2.0, 1.0, 1.0, 0.75, 1.0, 1.0, 1.0, 1.0, 1.5, 1.0]
    batch, w, X, dY = synth.random_case(1000 + r, in_f, out_f, r, 5, MIXED_LENGTHS, MIXED_MODES, slots, scale)
    res = run_smlm(batch, w, X, dY)
    assert res.plan_fwd == plan_oracle.forward_plan(batch.offsets, batch.slots, batch.modes)
    assert res.plan_bwd == plan_oracle.backward_plan(batch.offsets, batch.slots, batch.modes)
    _check(res, batch, w, X, dY, BF16_TOL)


@pytest.mark.parametrize("l_long", [1, 16, 1000])
def test_bf16_path_choice(l_long):
    """All-long, mostly-long and all-short decompositions all match the oracle."""
    batch, w, X, dY = synth.random_case(77, 192, 256, 16, 5, MIXED_LENGTHS, MIXED_MODES)
    res = run_smlm(batch, w, X, dY, l_long=l_long)
    _check(res, batch, w, X, dY, BF16_TOL)


def test_bf16_inplace_base_and_no_vsave():
    batch, w, X, dY = synth.random_case(5, 256, 256, 16, 5, MIXED_LENGTHS, MIXED_MODES)
    base = (X.float() @ w.W.float().T).to(torch.bfloat16)
    res = run_smlm(batch, w, X, dY, w_null=True, base_in=base, vsave=False)
    _check(res, batch, w, X, dY, BF16_TOL, base_in=base, w_null=True, check_v=False)


def test_bf16_accumulate_mask_and_no_dx():
    batch, w, X, dY = synth.random_case(6, 256, 192, 16, 5, MIXED_LENGTHS, MIXED_MODES)
    dA0 = torch.randn(5, 16, 256)
    dB0 = torch.randn(5, 192, 16)
    grads = [1, 0, 1, 1, 0]
    res = run_smlm(batch, w, X, dY, accumulate=True, dA0=dA0, dB0=dB0, grads=grads, want_dx=False)
    _, _, _, dA, dB = _oracle_all(batch, w, X, dY)
    rs, ft = batch.row_slot(), batch.ft_rows()
    for a in range(5):
        has_ft = np.any(rs[ft] == a)
        if grads[a] and has_ft:
            assert parity_err(res.dA[a].double() - dA0[a].double(), dA[a]) <= BF16_TOL
            assert parity_err(res.dB[a].double() - dB0[a].double(), dB[a]) <= BF16_TOL
        else:
            assert torch.equal(res.dA[a], dA0[a]) and torch.equal(res.dB[a], dB0[a])


def test_bf16_b_zero_identical_to_base_only():
    batch, w, X, dY = synth.random_case(8, 256, 256, 16, 5, MIXED_LENGTHS, MIXED_MODES)
    wz = synth.Weights(w.W, w.A, [torch.zeros_like(b) for b in w.B], w.slot_scale)
    r1 = run_smlm(batch, wz, X, dY, backward=False)
    nb = synth.Batch(batch.offsets, np.full_like(batch.slots, -1), batch.modes, None)
    r2 = run_smlm(nb, wz, X, dY, backward=False)
    assert torch.equal(r1.Y.float(), r2.Y.float())  # value equality (-0 == +0)
    ref = X.double() @ w.W.double().T
    assert parity_err(r1.Y, ref) <= BF16_TOL


def test_bf16_permutation_bit_exact():
    lengths = [300, 5, 1, 1, 64, 2, 130, 63, 1, 200]
    modes = [FINETUNE, DECODE, DECODE, DECODE, EVAL, DECODE, FINETUNE, PREFILL, DECODE, PREFILL]
    slots = [0, 1, 2, 1, 3, -1, 2, 3, 4, -1]
    batch, w, X, dY = synth.random_case(9, 256, 320, 16, 5, lengths, modes, slots)
    r1 = run_smlm(batch, w, X, dY)
    perm = [6, 2, 0, 9, 4, 1, 8, 3, 7, 5]
    rows = np.concatenate([np.arange(batch.offsets[g], batch.offsets[g + 1]) for g in perm])
    pb = synth.batch_from_lengths([lengths[g] for g in perm], [slots[g] for g in perm], [modes[g] for g in perm])
    r2 = run_smlm(pb, w, X[rows], dY[rows])
    assert torch.equal(r2.Y.float(), r1.Y[rows].float())
    ft = batch.ft_rows()
    pft = pb.ft_rows()
    assert torch.equal(r2.dX[pft].float(), r1.dX[rows][pft].float())
    for a in range(5):
        assert parity_err(r2.dA[a], r1.dA[a].double()) <= 1e-5 or (torch.all(r1.dA[a] == 0) and torch.all(r2.dA[a] == 0))


def test_bf16_dy_zero_and_determinism():
    batch, w, X, dY = synth.random_case(10, 256, 192, 16, 5, MIXED_LENGTHS, MIXED_MODES)
    r0 = run_smlm(batch, w, X, torch.zeros_like(dY))
    assert torch.all(r0.dA == 0) and torch.all(r0.dB == 0) and torch.all(r0.dX == 0)
    r1 = run_smlm(batch, w, X, dY)
    r2 = run_smlm(batch, w, X, dY)
    assert torch.equal(r1.dA, r2.dA) and torch.equal(r1.dB, r2.dB) and torch.equal(r1.Y, r2.Y)


def test_empty_batch():
    batch = synth.batch_from_lengths([], [], [])
    w = synth.draw_weights(torch.Generator().manual_seed(0), 64, 64, 16, 1)
    X = torch.zeros(0, 64, dtype=torch.bfloat16)
    res = run_smlm(batch, w, X, torch.zeros(0, 64, dtype=torch.bfloat16))
    assert res.Y.shape == (0, 64)


# ------------------------------------------------------------------------------------------
# full BASELINE.json shapes, sampled rows (plus exact-property checks at full size)
# ------------------------------------------------------------------------------------------
def _full_case(k, proj, rank=0):
    batch = synth.config_batch(k, rank)
    w = synth.config_weights(k, proj)
    X, dY = synth.config_activations(k, proj, batch.S, rank)
    return batch, w, X, dY


@pytest.mark.parametrize("k,proj", [(2, "q"), (2, "k"), (3, "down"), (4, "gate"), (4, "v")])
def test_full_config_sampled(k, proj):
    batch, w, X, dY = _full_case(k, proj)
    res = run_smlm(batch, w, X, dY)
    rows = synth.sample_rows(batch, every=97)
    _check(res, batch, w, X, dY, BF16_TOL, rows=rows)
    # Euler identities at full size (no oracle): <dA_a, A_a> = <dB_a, B_a> = <dY, Y_lora_a>
    if len(batch.ft_rows()):
        rs, ft = batch.row_slot(), batch.ft_rows()
        for a in sorted(set(rs[ft].tolist())):
            if a < 0:
                continue
            lhsA = float((res.dA[a].double() * w.A[a].double()).sum())
            lhsB = float((res.dB[a].double() * w.B[a].double()).sum())
            assert abs(lhsA - lhsB) <= 2e-2 * (abs(lhsA) + abs(lhsB))


@pytest.mark.parametrize("rows,in_f,out_f,r", [(200, 512, 320, 16), (64, 1024, 256, 8), (450, 512, 192, 32),
                                               (300, 192, 256, 16), (512, 1024, 128, 64), (384, 14336, 256, 16)])
def test_bf16_decode_batches(rows, in_f, out_f, r):
    """Pure decode batches (the transposed split-K kernel path): one-row DECODE segments, random
    slots including base-only rows, unsorted."""
    g = torch.Generator().manual_seed(rows + in_f)
    slots = torch.randint(-1, 6, (rows,), generator=g).tolist()
    batch, w, X, dY = synth.random_case(rows * 7 + r, in_f, out_f, r, 6, [1] * rows, [DECODE] * rows, slots)
    res = run_smlm(batch, w, X, dY, backward=False)
    assert res.plan_fwd == plan_oracle.forward_plan(batch.offsets, batch.slots, batch.modes)
    Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    assert parity_err(res.Y, Y) <= BF16_TOL


def test_bf16_decode_many_adapters_unsorted():
    """512 unsorted one-row requests over 64 adapters (two 256-row groups, up to 8 adapters per
    32-column expand split, several shrink items per adapter)."""
    g = torch.Generator().manual_seed(64)
    rows = 512
    slots = torch.randint(-1, 64, (rows,), generator=g).tolist()
    modes = [DECODE if i % 17 else FINETUNE for i in range(rows)]
    batch, w, X, dY = synth.random_case(640, 1024, 512, 16, 64, [1] * rows, modes, slots)
    res = run_smlm(batch, w, X, dY, backward=False)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    assert parity_err(res.Y, Y) <= BF16_TOL
    ft = batch.ft_rows()
    ft = ft[batch.row_slot()[ft] >= 0]
    assert parity_err(res.V.double().numpy()[ft], V[ft]) <= BF16_TOL


def test_bf16_decode_grouped_with_finetune_short_rows():
    """Short fine-tune segments inside a pure-short batch: V_save and the backward still match."""
    lengths = [3, 1, 5, 1, 2, 7, 1, 1]
    modes = [FINETUNE, DECODE, FINETUNE, DECODE, EVAL, FINETUNE, DECODE, PREFILL]
    batch, w, X, dY = synth.random_case(31, 1024, 384, 16, 4, lengths, modes, [0, 1, 2, 1, 3, 0, -1, 2])
    res = run_smlm(batch, w, X, dY)
    _check(res, batch, w, X, dY, BF16_TOL)


@pytest.mark.parametrize("ks", [1, 2, 3, 8, -1, 0])
def test_bf16_decode_ksplit_variants(ks):
    """The single-launch decode kernel (kernels_dec3.cu) at forced split-K factors (pool option
    SMLM_OPT_DEC_KSPLIT): every split count matches the oracle (in-kernel reduce-scatter of the
    fp32 partials); ks = -1 runs the same batch through the mixed-batch path instead
    (SMLM_OPT_DECODE_KERNEL = 0); ks = 0 is the automatic split with a cooperative launch
    (SMLM_OPT_DEC_COOPERATIVE)."""
    from paper_2511_00101_b200 import smlm as S
    opts = ({S.SMLM_OPT_DECODE_KERNEL: 0} if ks < 0 else
            {S.SMLM_OPT_DEC_COOPERATIVE: 1} if ks == 0 else {S.SMLM_OPT_DEC_KSPLIT: ks})
    g = torch.Generator().manual_seed(5)
    rows = 200
    slots = torch.randint(-1, 6, (rows,), generator=g).tolist()
    modes = [DECODE] * (rows - 3) + [FINETUNE] * 3
    batch, w, X, dY = synth.random_case(77, 1024, 640, 16, 6, [1] * rows, modes, slots)
    res = run_smlm(batch, w, X, dY, backward=False, options=opts)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    assert parity_err(res.Y, Y) <= BF16_TOL
    ft = batch.ft_rows()
    ft = ft[batch.row_slot()[ft] >= 0]
    assert parity_err(res.V.double().numpy()[ft], V[ft]) <= BF16_TOL


def test_bf16_decode_b_zero_and_permutation():
    """Pure decode batch: B = 0 is value-identical to all slots -1 (the split-K ranges do not
    depend on the adapters; the expand adds exact zeros), and permuting the one-row segments
    permutes Y bit-exactly (per-row arithmetic is position independent)."""
    rows = 240
    g = torch.Generator().manual_seed(11)
    slots = torch.randint(-1, 7, (rows,), generator=g).tolist()
    batch, w, X, dY = synth.random_case(12, 1024, 768, 16, 7, [1] * rows, [DECODE] * rows, slots)
    wz = synth.Weights(w.W, w.A, [torch.zeros_like(b) for b in w.B], w.slot_scale)
    r1 = run_smlm(batch, wz, X, dY, backward=False)
    nb = synth.Batch(batch.offsets, np.full_like(batch.slots, -1), batch.modes, None)
    r2 = run_smlm(nb, wz, X, dY, backward=False)
    assert torch.equal(r1.Y.float(), r2.Y.float())
    r3 = run_smlm(batch, w, X, dY, backward=False)
    perm = torch.randperm(rows, generator=g).numpy()
    pb = synth.batch_from_lengths([1] * rows, [slots[i] for i in perm], [DECODE] * rows)
    r4 = run_smlm(pb, w, X[perm], dY[perm], backward=False)
    assert torch.equal(r4.Y.float(), r3.Y[perm].float())


def _multi_case(seed, in_f, outs, r, U, rows, ft_rows=3):
    g = torch.Generator().manual_seed(seed)
    slots = torch.randint(-1, U, (rows,), generator=g).tolist()
    modes = [DECODE] * (rows - ft_rows) + [FINETUNE] * ft_rows
    cases = [synth.random_case(seed * 10 + i, in_f, o, r, U, [1] * rows, modes, slots) for i, o in enumerate(outs)]
    return cases[0][0], [c[1] for c in cases], cases[0][2]


def _run_multi(batch, ws_, X, slot_scales=None):
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    in_f, r, U = X.shape[1], ws_[0].A[0].shape[0], len(ws_[0].A)
    pools, keep = [], []
    for i, w in enumerate(ws_):
        pool = S.Pool(in_f, w.W.shape[0], r, U)
        for a in range(U):
            A, B = w.A[a].to(dev).contiguous(), w.B[a].to(dev).contiguous()
            sc = w.slot_scale[a] if slot_scales is None else slot_scales[i][a]
            assert pool.register(A, B, sc) == a
        pools.append(pool)
    b = S.Batch.from_synth(batch)
    Xd = X.to(dev).contiguous()
    Ws = [w.W.to(dev).contiguous() for w in ws_]
    Ys = [torch.full((batch.S, w.W.shape[0]), float("nan"), dtype=torch.bfloat16, device=dev) for w in ws_]
    Vs = [torch.zeros(batch.S, r, dtype=torch.bfloat16, device=dev) for _ in ws_]
    n = S.smlm_workspace_size_multi([p.h for p in pools], b)
    wsb = torch.empty(max(n, 256), dtype=torch.uint8, device=dev)
    n0 = S.smlm_launch_count()
    S.smlm_forward_multi([p.h for p in pools], b, Xd, Ws, Ys, Vs, wsb)
    torch.cuda.synchronize()
    launches = S.smlm_launch_count() - n0
    for p in pools:
        p.close()
    return [y.cpu() for y in Ys], [v.cpu() for v in Vs], launches


@pytest.mark.parametrize("rows,in_f,outs,r", [(256, 1024, (1024, 256, 256), 16), (200, 512, (320, 192), 8),
                                              (450, 512, (256, 128, 384, 64), 32), (64, 192, (128,), 64)])
def test_bf16_decode_multi_projection(rows, in_f, outs, r):
    """smlm_forward_multi: several projections sharing X in ONE launch, each Y and V_save against
    the oracle of its own projection."""
    batch, ws_, X = _multi_case(rows + in_f, in_f, outs, r, 5, rows)
    Ys, Vs, launches = _run_multi(batch, ws_, X)
    assert launches == 1
    ft = batch.ft_rows()
    ft = ft[batch.row_slot()[ft] >= 0]
    for i, w in enumerate(ws_):
        Yr, Vr = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
        assert parity_err(Ys[i], Yr) <= BF16_TOL, i
        if len(ft):
            assert parity_err(Vs[i].double().numpy()[ft], Vr[ft]) <= BF16_TOL, i


def test_bf16_multi_fallbacks_and_errors():
    """Different slot scales across pools -> per-pool calls (still correct); a mixed batch with
    long segments -> per-pool calls; a slot missing from one pool -> SMLM_E_SLOT."""
    from paper_2511_00101_b200 import smlm as S
    batch, ws_, X = _multi_case(3, 512, (256, 192), 16, 4, 100)
    scales = [[2.0] * 4, [1.0, 2.0, 3.0, 0.5]]
    Ys, _, launches = _run_multi(batch, ws_, X, slot_scales=scales)
    assert launches >= 2
    for i, w in enumerate(ws_):
        Yr, _ = oracle.forward(batch, w.W, w.A, w.B, scales[i], X)
        assert parity_err(Ys[i], Yr) <= BF16_TOL
    lengths = [130, 1, 1, 70, 2]
    modes = [PREFILL, DECODE, DECODE, EVAL, DECODE]
    cases = [synth.random_case(40 + i, 256, o, 16, 3, lengths, modes, [0, 1, 2, -1, 1]) for i, o in enumerate((256, 128))]
    Ys, _, _ = _run_multi(cases[0][0], [c[1] for c in cases], cases[0][2])
    for i, c in enumerate(cases):
        Yr, _ = oracle.forward(c[0], c[1].W, c[1].A, c[1].B, c[1].slot_scale, cases[0][2])
        assert parity_err(Ys[i], Yr) <= BF16_TOL
    p0, p1 = S.Pool(256, 256, 16, 4), S.Pool(256, 128, 16, 4)
    A, B0, B1 = (torch.zeros(16, 256, dtype=torch.bfloat16, device="cuda"),
                 torch.zeros(256, 16, dtype=torch.bfloat16, device="cuda"),
                 torch.zeros(128, 16, dtype=torch.bfloat16, device="cuda"))
    p0.register(A, B0, 2.0)
    p0.register(A, B0, 2.0)
    p1.register(A, B1, 2.0)
    b = S.Batch([0, 1, 2], [0, 1], [DECODE, DECODE])
    with pytest.raises(S.SmlmError) as ei:
        S.smlm_workspace_size_multi([p0.h, p1.h], b) or S.smlm_forward_multi(
            [p0.h, p1.h], b, torch.zeros(2, 256, dtype=torch.bfloat16, device="cuda"), [None, None], [None, None])
    assert ei.value.code in (S.SMLM_E_SLOT, S.SMLM_E_INVALID)
    p0.close()
    p1.close()


def test_bf16_decode_graph_capture_replays_eager():
    """A decode call recorded into a CUDA graph (inline plan in the kernel parameters) replays to
    the same Y as the eager call, bit for bit, including after the inputs change in place."""
    from paper_2511_00101_b200 import smlm as S
    batch, ws_, X = _multi_case(21, 512, (256, 128), 16, 4, 96)
    dev = torch.device("cuda", 0)
    pools = []
    for w in ws_:
        pool = S.Pool(512, w.W.shape[0], 16, 4)
        for a in range(4):
            pool.register(w.A[a].to(dev).contiguous(), w.B[a].to(dev).contiguous(), w.slot_scale[a])
        pools.append(pool)
    b = S.Batch.from_synth(batch)
    Xd = X.to(dev).contiguous()
    Ws = [w.W.to(dev).contiguous() for w in ws_]
    Ys = [torch.empty(batch.S, w.W.shape[0], dtype=torch.bfloat16, device=dev) for w in ws_]
    wsb = torch.empty(S.smlm_workspace_size_multi([p.h for p in pools], b) + 256, dtype=torch.uint8, device=dev)
    S.smlm_forward_multi([p.h for p in pools], b, Xd, Ws, Ys, None, wsb)
    torch.cuda.synchronize()
    eager = [y.clone() for y in Ys]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        S.smlm_forward_multi([p.h for p in pools], b, Xd, Ws, Ys, None, wsb)
    for y in Ys:
        y.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    for y, e in zip(Ys, eager):
        assert torch.equal(y, e)
    Xd.mul_(-1)                                   # new inputs, same buffers: Y flips sign exactly
    g.replay()
    torch.cuda.synchronize()
    for y, e in zip(Ys, eager):
        assert torch.equal(y.float(), -e.float())
    for p in pools:
        p.close()


@pytest.mark.parametrize("rows,n_ad,outs", [(256, 160, (512,)), (1, 4, (256, 128)), (512, 64, (512, 256, 256))])
def test_bf16_decode_edge_shapes(rows, n_ad, outs):
    """Decode edge cases: many adapters (13 stacked-A tiles), a single row, and 512 rows x 3
    projections x 64 adapters (split factors drop to 1)."""
    batch, ws_, X = _multi_case(rows * 3 + n_ad, 512, outs, 16, n_ad, rows, ft_rows=min(3, rows))
    Ys, Vs, launches = _run_multi(batch, ws_, X)
    assert launches == 1
    ft = batch.ft_rows()
    ft = ft[batch.row_slot()[ft] >= 0]
    for i, w in enumerate(ws_):
        Yr, Vr = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
        assert parity_err(Ys[i], Yr) <= BF16_TOL, i
        if len(ft):
            assert parity_err(Vs[i].double().numpy()[ft], Vr[ft]) <= BF16_TOL, i


# ------------------------------------------------------------------------------------------
# heterogeneous ranks in one pool: adapters registered with their own rank
# ------------------------------------------------------------------------------------------
def _truncate_ranks(w, ranks):
    w.A = [a[:ra].contiguous() for a, ra in zip(w.A, ranks)]
    w.B = [b[:, :ra].contiguous() for b, ra in zip(w.B, ranks)]
    return w


@pytest.mark.parametrize("r,ranks", [(16, [16, 8, 16, 8, 8]), (64, [64, 8, 32, 24, 48]), (32, [8, 32, 16, 24, 32])])
def test_bf16_mixed_heterogeneous_ranks(r, ranks):
    """Mixed batch (long fine-tune/prefill/eval tiles + short decode rows), forward and backward:
    parity with the oracle (which zero-pads to the pool rank, an exact identity pinned in
    test_oracle_pins), and no gradient write past an adapter's own rank (guards in run_smlm)."""
    slots = [0, 1, 2, 1, 3, -1, 2, 0, 3, 4, -1, 4, 0]
    batch, w, X, dY = synth.random_case(3000 + r, 256, 320, r, 5, MIXED_LENGTHS, MIXED_MODES, slots)
    w = _truncate_ranks(w, ranks)
    res = run_smlm(batch, w, X, dY)
    _check(res, batch, w, X, dY, BF16_TOL)


@pytest.mark.parametrize("rows,r,ranks", [(256, 16, [8, 16, 8, 16, 8, 16]), (300, 64, [8, 16, 24, 32, 48, 64])])
def test_bf16_decode_heterogeneous_ranks(rows, r, ranks):
    """Pure decode batch (the single-launch decode kernel) with adapters of different ranks."""
    g = torch.Generator().manual_seed(rows + r)
    slots = torch.randint(-1, 6, (rows,), generator=g).tolist()
    batch, w, X, dY = synth.random_case(rows * 3 + r, 1024, 512, r, 6, [1] * rows, [DECODE] * rows, slots)
    w = _truncate_ranks(w, ranks)
    res = run_smlm(batch, w, X, dY, backward=False)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
    assert parity_err(res.Y, Y) <= BF16_TOL


def test_bf16_lower_rank_equals_zero_padded_bitwise():
    """A rank-8 adapter in a rank-16 pool gives bit for bit the result of the same adapter
    zero-padded to rank 16 and registered at the pool rank (forward, V_save, dX, dA, dB)."""
    batch, w, X, dY = synth.random_case(91, 256, 192, 16, 3, MIXED_LENGTHS, MIXED_MODES,
                                        [0, 1, 2, 1, 0, -1, 2, 0, 1, 2, -1, 0, 1])
    low = _truncate_ranks(synth.random_case(91, 256, 192, 16, 3, [1], [DECODE], [0])[1], [8, 16, 8])
    pad = synth.random_case(91, 256, 192, 16, 3, [1], [DECODE], [0])[1]
    for a in (0, 2):
        pad.A[a] = torch.cat([low.A[a], torch.zeros_like(low.A[a])])
        pad.B[a] = torch.cat([low.B[a], torch.zeros_like(low.B[a])], dim=1)
    low.W = pad.W = w.W
    r_low = run_smlm(batch, low, X, dY)
    r_pad = run_smlm(batch, pad, X, dY)
    assert torch.equal(r_low.Y, r_pad.Y) and torch.equal(r_low.V, r_pad.V) and torch.equal(r_low.dX, r_pad.dX)
    assert torch.equal(r_low.dA, r_pad.dA) and torch.equal(r_low.dB, r_pad.dB)


def test_register_rank_errors():
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    pool = S.Pool(128, 128, 16, 4, S.SMLM_BF16, 0)
    for ra in (12, 32, 4):   # not a multiple of 8 / above the pool rank / below 8
        A = torch.zeros(ra, 128, dtype=torch.bfloat16, device=dev)
        B = torch.zeros(128, ra, dtype=torch.bfloat16, device=dev)
        with pytest.raises(S.SmlmError) as e:
            S.smlm_adapter_register_rank(pool.h, A, B, ra, 1.0)
        assert e.value.code == S.SMLM_E_SHAPE
    pool.close()
    pf = S.Pool(128, 128, 16, 4, S.SMLM_FP32, 0)
    with pytest.raises(S.SmlmError) as e:
        S.smlm_adapter_register_rank(pf.h, torch.zeros(8, 128, device=dev), torch.zeros(128, 8, device=dev), 8, 1.0)
    assert e.value.code == S.SMLM_E_SHAPE
    pf.close()


def test_bf16_large_plan_memcpy_fallback():
    """A batch whose plan exceeds one kernel-parameter block (3000 one-row decode segments of 40
    adapters plus a fine-tune segment: > 32 KB of plan records) takes the pinned-ring memcpy
    upload instead of the parameter copy kernel; parity as usual."""
    rows = 3000
    g = torch.Generator().manual_seed(17)
    slots = torch.randint(-1, 40, (rows,), generator=g).tolist() + [3]
    lengths = [1] * rows + [200]
    modes = [DECODE] * rows + [FINETUNE]
    batch, w, X, dY = synth.random_case(4321, 256, 192, 16, 40, lengths, modes, slots)
    res = run_smlm(batch, w, X, dY)
    rows_chk = np.concatenate([np.arange(0, rows, 7), np.arange(rows, rows + 200)])
    _check(res, batch, w, X, dY, BF16_TOL, rows=rows_chk)


@pytest.mark.parametrize("r,outs", [(16, (320, 192, 192)), (32, (256, 512)), (64, (192, 256)), (16, (128, 256, 192, 320)),
                                    (64, (192, 256, 128))])   # last: 3 x 64 > 128 columns -> per-pool calls
def test_bf16_mixed_multi_projection(r, outs):
    """Mixed batch through smlm_forward_multi (f1 for mixed batches): one shared pre-shrink pass
    for all projections, then each projection's GEMM.  Every projection matches the oracle (Y on
    all rows, V_save on fine-tune rows) and is bit-identical to its own smlm_forward call."""
    slots = [0, 1, 2, 1, 3, -1, 2, 0, 3, 4, -1, 4, 0]
    cases = [synth.random_case(5000 + 10 * r + i, 256, o, r, 5, MIXED_LENGTHS, MIXED_MODES, slots)
             for i, o in enumerate(outs)]
    batch, X = cases[0][0], cases[0][2]
    ws_ = [c[1] for c in cases]
    Ys, Vs, launches = _run_multi(batch, ws_, X)
    ft = batch.ft_rows()
    rs = batch.row_slot()
    ft_lora = ft[rs[ft] >= 0]
    for i, w in enumerate(ws_):
        Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X)
        assert parity_err(Ys[i], Y) <= BF16_TOL, i
        assert parity_err(Vs[i].double().numpy()[ft_lora], V[ft_lora]) <= BF16_TOL, i
        single = run_smlm(batch, w, X, None, backward=False)
        assert torch.equal(single.Y, Ys[i]), f"projection {i}: multi differs from the single call"
        assert torch.equal(single.V[ft_lora], Vs[i][ft_lora]), i


def test_full_c4_qkv_multi_sampled():
    """C4 (unified batch, full size) q/k/v through smlm_forward_multi: the shared pre-shrink at
    13 448 rows and 64 adapters, checked on sampled rows of every projection."""
    batch = synth.config_batch(4)
    ws_ = [synth.config_weights(4, p) for p in ("q", "k", "v")]
    X, _ = synth.config_activations(4, "q", batch.S)
    Ys, Vs, launches = _run_multi(batch, ws_, X)
    rows = synth.sample_rows(batch, every=97)
    for i, w in enumerate(ws_):
        Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, rows=rows)
        assert parity_err(Ys[i].double().numpy()[rows], Y[rows]) <= BF16_TOL, i


@pytest.mark.parametrize("r,outs,lengths", [
    (16, (320, 192, 192), [300, 260, 3, 1, 140]),          # q/k/v-like: three projections
    (32, (256, 512), [129, 127, 1, 2, 513]),               # gate/up-like, odd tile counts
    (64, (192,), [200, 70]),
])
def test_bf16_backward_multi_equals_single(r, outs, lengths):
    """smlm_backward_multi (one dX GEMM launch over every projection's n-tiles) is bit-identical to
    the per-projection smlm_backward calls and matches the oracle."""
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    in_f, U = 256, 5
    modes = [FINETUNE, FINETUNE, DECODE, DECODE, FINETUNE][:len(lengths)]
    slots = [0, 3, 1, -1, 2][:len(lengths)]
    batch = synth.batch_from_lengths(lengths, slots, modes)
    g = torch.Generator().manual_seed(77)
    ws_ = [synth.draw_weights(g, in_f, o, r, U) for o in outs]
    X = torch.randn(batch.S, in_f, generator=g).to(torch.bfloat16)
    dYs = [torch.randn(batch.S, o, generator=g).to(torch.bfloat16) for o in outs]
    b = S.Batch.from_synth(batch)
    Xd = X.to(dev)

    def run(multi):
        pools, keep, grads = [], [], []
        for w in ws_:
            pool = S.Pool(in_f, w.W.shape[0], r, U)
            gA = torch.zeros(U, r, in_f, device=dev)
            gB = torch.zeros(U, w.W.shape[0], r, device=dev)
            for a in range(U):
                A, B = w.A[a].to(dev).contiguous(), w.B[a].to(dev).contiguous()
                keep += [A, B]
                pool.register(A, B, w.slot_scale[a])
                pool.set_grad(a, gA[a], gB[a])
            pools.append(pool)
            grads.append((gA, gB))
        Wd = [w.W.to(dev) for w in ws_]
        dYd = [y.to(dev) for y in dYs]
        dXs = [torch.zeros(batch.S, in_f, dtype=torch.bfloat16, device=dev) for _ in ws_]
        Vs = []
        for i, pool in enumerate(pools):
            V = torch.zeros(batch.S, r, dtype=torch.bfloat16, device=dev)
            pool.forward(b, Xd, Wd[i], V_save=V)
            Vs.append(V)
        if multi:
            n0 = S.smlm_launch_count()
            ws = torch.empty(S.smlm_workspace_size_backward_multi([p.h for p in pools], b) + 256, dtype=torch.uint8,
                             device=dev)
            S.smlm_backward_multi([p.h for p in pools], b, Xd, Wd, dYd, Vs, dXs, ws=ws)
        else:
            for i, pool in enumerate(pools):
                pool.backward(b, Xd, Wd[i], dYd[i], Vs[i], dXs[i])
        torch.cuda.synchronize()
        for p_ in pools:
            p_.close()
        return [x.cpu() for x in dXs], [(a.cpu(), bb.cpu()) for a, bb in grads]

    dX1, g1 = run(False)
    dXm, gm = run(True)
    ft = batch.ft_rows()
    rs = batch.row_slot()
    for i, w in enumerate(ws_):
        assert torch.equal(dX1[i][ft], dXm[i][ft]), i
        assert torch.equal(g1[i][0], gm[i][0]) and torch.equal(g1[i][1], gm[i][1]), i
        dXr, dAr, dBr = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dYs[i])
        assert parity_err(dXm[i].double().numpy()[ft], dXr[ft]) <= BF16_TOL, i
        for a in sorted(set(rs[ft].tolist()) - {-1}):
            assert parity_err(gm[i][0][a], dAr[a]) <= BF16_TOL, (i, a)
            assert parity_err(gm[i][1][a], dBr[a]) <= BF16_TOL, (i, a)
