"""GPU parity of LoRA dropout on the fine-tune rows (App. D Table 5
lora_dropout 0.05; R13) against the fp64 oracle, which takes the keep mask as an explicit
input: the mask comes from synth.dropout_keep (the counter-based generator) and the CUDA path draws
the same bits from (seed, row, column) with its own implementation of the hash -- the two agree
only if the kernels apply dropout exactly where the definition says (x feeding A_a of FINETUNE
rows: the pre-shrink, the short-row shrink, the dX LoRA term, the dA contraction, V recompute).

Bars: bf16 2e-2, fp32 test mode 1e-5 (tests/util.py); p = 0 is bit-identical to no dropout."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import DECODE, EVAL, FINETUNE, PREFILL
from tests.smlm_run import run_smlm
from tests.util import BF16_TOL, FP32_TOL, parity_err

pytestmark = pytest.mark.gpu

GOLDEN = 0x9E3779B97F4A7C15


def _check(res, batch, w, X, dY, p, seed, tol, vsave=True, has_dx=True):
    keep = synth.dropout_keep(seed, p, batch.S, X.shape[1])
    pe = synth.dropout_effective_p(p)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, keep=keep, p=pe)
    dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, keep=keep, p=pe)
    errs = {"Y": parity_err(res.Y, Y)}
    ft = batch.ft_rows()
    rs = batch.row_slot()
    ftl = ft[rs[ft] >= 0]
    if vsave and len(ftl):
        errs["V"] = parity_err(res.V.double().numpy()[ftl], V[ftl])
    if has_dx and len(ft):
        errs["dX"] = parity_err(res.dX.double().numpy()[ft], dX[ft])
    for a in sorted(set(rs[ft].tolist()) - {-1}):
        errs[f"dA{a}"] = parity_err(res.dA[a], dA[a])
        errs[f"dB{a}"] = parity_err(res.dB[a], dB[a])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (bad, errs)
    return errs


@pytest.mark.parametrize("p", [0.05, 0.3])
@pytest.mark.parametrize("case", ["mixed", "short_ft", "odd_tiles"])
def test_bf16_dropout_parity(p, case):
    if case == "mixed":      # long FT tiles (pre-shrink, CTA-pair dX), short FT rows (SIMT shrink), others
        lengths, modes, slots = [300, 3, 1, 70, 2, 130], [FINETUNE, FINETUNE, DECODE, PREFILL, EVAL, FINETUNE], \
            [0, 1, 2, 3, 1, 2]
    elif case == "short_ft":  # a pure-short batch with fine-tune rows: not the decode kernel (mask)
        lengths, modes, slots = [3, 1, 5, 1, 2], [FINETUNE, DECODE, FINETUNE, DECODE, EVAL], [0, 1, 2, 1, 3]
    else:                     # FT tiles paired across segments / adapters, a base-only FT segment
        lengths, modes, slots = [129, 127, 255, 64], [FINETUNE, FINETUNE, FINETUNE, FINETUNE], [0, 1, -1, 0]
    batch, w, X, dY = synth.random_case(61, 512, 384, 16, 4, lengths, modes, slots)
    seed = 0x1234_5678_9ABC_DEF0
    res = run_smlm(batch, w, X, dY, dropout=(p, seed))
    _check(res, batch, w, X, dY, p, seed, BF16_TOL)


def test_bf16_dropout_recompute_v_and_accumulate():
    """Backward without V_save (V recomputed from x with the same mask) and accumulate = 1."""
    lengths, modes, slots = [200, 4, 90], [FINETUNE, FINETUNE, PREFILL], [0, 1, 2]
    batch, w, X, dY = synth.random_case(62, 256, 320, 32, 3, lengths, modes, slots)
    p, seed = 0.1, 77
    res = run_smlm(batch, w, X, dY, dropout=(p, seed), vsave=False)
    _check(res, batch, w, X, dY, p, seed, BF16_TOL, vsave=False)


def test_fp32_dropout_parity():
    lengths, modes, slots = [12, 8, 8, 4], [FINETUNE, EVAL, PREFILL, FINETUNE], [0, 1, 2, 0]
    batch, w, X, dY = synth.random_case(63, 64, 48, 4, 3, lengths, modes, slots, dtype=torch.float32)
    p, seed = 0.25, 4242
    res = run_smlm(batch, w, X, dY, dropout=(p, seed))
    _check(res, batch, w, X, dY, p, seed, FP32_TOL)


def test_dropout_p0_bit_identical_and_mask_changes_with_seed():
    lengths, modes, slots = [300, 3, 1, 70], [FINETUNE, FINETUNE, DECODE, PREFILL], [0, 1, 2, 3]
    batch, w, X, dY = synth.random_case(64, 512, 256, 16, 4, lengths, modes, slots)
    r0 = run_smlm(batch, w, X, dY)
    r1 = run_smlm(batch, w, X, dY, dropout=(0.0, 999))
    for a, b in ((r0.Y, r1.Y), (r0.V, r1.V), (r0.dX, r1.dX), (r0.dA, r1.dA), (r0.dB, r1.dB)):
        assert torch.equal(a, b)
    ra = run_smlm(batch, w, X, dY, dropout=(0.05, 1))
    rb = run_smlm(batch, w, X, dY, dropout=(0.05, 2))
    ft = batch.ft_rows()
    assert not torch.equal(ra.Y[ft], rb.Y[ft])
    other = np.setdiff1d(np.arange(batch.S), ft)
    assert torch.equal(ra.Y[other], rb.Y[other]) and torch.equal(ra.Y[other], r0.Y[other])


def test_dropout_multi_projection_independent_masks():
    """smlm_forward_multi / smlm_backward_multi with dropout: projection i draws its mask with seed
    + i * 0x9E3779B97F4A7C15 (PEFT: one dropout module per LoRA layer)."""
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    lengths, modes, slots = [260, 2, 130], [FINETUNE, DECODE, FINETUNE], [0, 1, 2]
    batch = synth.batch_from_lengths(lengths, slots, modes)
    g = torch.Generator().manual_seed(65)
    outs = (256, 192)
    ws_ = [synth.draw_weights(g, 512, o, 16, 3) for o in outs]
    X = torch.randn(batch.S, 512, generator=g).to(torch.bfloat16)
    dYs = [torch.randn(batch.S, o, generator=g).to(torch.bfloat16) for o in outs]
    p, seed = 0.2, 31337
    b = S.Batch.from_synth(batch, p, seed)
    pools, keep, grads = [], [], []
    for w in ws_:
        pool = S.Pool(512, w.W.shape[0], 16, 3)
        gA = torch.zeros(3, 16, 512, device=dev)
        gB = torch.zeros(3, w.W.shape[0], 16, device=dev)
        for a in range(3):
            A, B = w.A[a].to(dev).contiguous(), w.B[a].to(dev).contiguous()
            keep += [A, B]
            pool.register(A, B, w.slot_scale[a])
            pool.set_grad(a, gA[a], gB[a])
        pools.append(pool)
        grads.append((gA, gB))
    hs = [q.h for q in pools]
    Xd = X.to(dev)
    Wd = [w.W.to(dev) for w in ws_]
    Ys = [torch.empty(batch.S, o, dtype=torch.bfloat16, device=dev) for o in outs]
    Vs = [torch.zeros(batch.S, 16, dtype=torch.bfloat16, device=dev) for _ in outs]
    dXs = [torch.zeros(batch.S, 512, dtype=torch.bfloat16, device=dev) for _ in outs]
    wsf = torch.empty(S.smlm_workspace_size_multi(hs, b) + 256, dtype=torch.uint8, device=dev)
    S.smlm_forward_multi(hs, b, Xd, Wd, Ys, Vs, wsf)
    wsb = torch.empty(S.smlm_workspace_size_backward_multi(hs, b) + 256, dtype=torch.uint8, device=dev)
    S.smlm_backward_multi(hs, b, Xd, Wd, [y.to(dev) for y in dYs], Vs, dXs, ws=wsb)
    torch.cuda.synchronize()
    ft = batch.ft_rows()
    for i, w in enumerate(ws_):
        si = (seed + i * GOLDEN) & 0xFFFFFFFFFFFFFFFF
        km = synth.dropout_keep(si, p, batch.S, 512)
        pe = synth.dropout_effective_p(p)
        Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, keep=km, p=pe)
        dX, dA, dB = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dYs[i], keep=km, p=pe)
        assert parity_err(Ys[i].cpu(), Y) <= BF16_TOL, i
        assert parity_err(dXs[i].cpu().double().numpy()[ft], dX[ft]) <= BF16_TOL, i
        for a in (0, 2):
            assert parity_err(grads[i][0][a].cpu(), dA[a]) <= BF16_TOL, (i, a)
            assert parity_err(grads[i][1][a].cpu(), dB[a]) <= BF16_TOL, (i, a)
    for q in pools:
        q.close()


def test_dropout_errors():
    from paper_2511_00101_b200 import smlm as S
    lengths, modes, slots = [200, 4], [FINETUNE, DECODE], [0, 1]
    batch, w, X, dY = synth.random_case(66, 256, 256, 16, 2, lengths, modes, slots)
    with pytest.raises(S.SmlmError) as e:
        run_smlm(batch, w, X, dY, dropout=(0.1, 1), options={S.SMLM_OPT_CTA_PAIR: 0})
    assert e.value.code == S.SMLM_E_UNSUPPORTED
    with pytest.raises(S.SmlmError) as e:
        run_smlm(batch, w, X, dY, dropout=(1.0, 1))
    assert e.value.code == S.SMLM_E_INVALID
    # no fine-tune rows: dropout has nothing to act on, any path is fine
    b2, w2, X2, dY2 = synth.random_case(67, 256, 256, 16, 2, [50, 3], [PREFILL, DECODE], [0, 1])
    r = run_smlm(b2, w2, X2, dY2, dropout=(0.5, 3), options={S.SMLM_OPT_CTA_PAIR: 0}, backward=False)
    Y, _ = oracle.forward(b2, w2.W, w2.A, w2.B, w2.slot_scale, X2)
    assert parity_err(r.Y, Y) <= BF16_TOL
