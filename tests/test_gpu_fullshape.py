"""Full BASELINE.json shapes (VERDICT r1 "close the full-shape parity gaps"): every projection's
backward at the C4 size (dX at N = 14336 for gate/up and K = 14336 for down), gate/up through
smlm_forward_multi at C4 size, the fused q/k/v decode launch at the C2 size (in = 4096, 32
adapters, 256 rows), the bench's exact step schedule (two-stream backward), and the full-size
Euler identities of SURVEY.md §8(c) pin 8 -- against the fp64 oracle on sampled rows (dA/dB over
ALL fine-tune rows), and against the identities on every fine-tune row.

Euler / bilinearity identities (no oracle, exact in real arithmetic; checked in fp64 on the GPU's
own outputs): for each fine-tune adapter a, over its fine-tune rows,
    <dA_a, A_a> = <dB_a, B_a> = <dY, Y - X W^T>       (Y is linear in A alone and in B alone)
and over all fine-tune rows  <dX, X> = <dY, Y>          (Y is linear in X).
Bound: |lhs - rhs| <= 2e-2 * sum of |terms| (bf16 rounding of Y, dX, s*V, s*U)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.smlm_run import run_smlm
from tests.util import BF16_TOL, parity_err

pytestmark = pytest.mark.gpu


def _full(k, proj):
    batch = synth.config_batch(k)
    w = synth.config_weights(k, proj)
    X, dY = synth.config_activations(k, proj, batch.S)
    return batch, w, X, dY


def _euler(batch, w, X, dY, Y, dX, dA, dB):
    """SURVEY §8(c) pin 8 on the GPU's outputs, fp64 (base product X W^T by torch on the GPU)."""
    dev = torch.device("cuda", 0)
    ft = batch.ft_rows()
    rs = batch.row_slot()
    Xf = X[ft].to(dev, torch.float64)
    base = Xf @ w.W.to(dev, torch.float64).T
    Yf = Y[ft].to(dev, torch.float64)
    dYf = dY[ft].to(dev, torch.float64)
    dXf = dX[ft].to(dev, torch.float64)
    # <dX, X> = <dY, Y> over every fine-tune row
    lhs = float((dXf * Xf).sum())
    rhs = float((dYf * Yf).sum())
    mag = float((dXf * Xf).abs().sum() + (dYf * Yf).abs().sum())
    assert abs(lhs - rhs) <= 2e-2 * mag, ("<dX,X> vs <dY,Y>", lhs, rhs, mag)
    for a in sorted(set(rs[ft].tolist())):
        if a < 0:
            continue
        sel = torch.from_numpy((rs[ft] == a)).to(dev)
        dly = ((Yf - base) * dYf)[sel]
        rhs = float(dly.sum())
        tA = dA[a].to(dev, torch.float64) * w.A[a].to(dev, torch.float64)
        tB = dB[a].to(dev, torch.float64) * w.B[a].to(dev, torch.float64)
        lhsA, lhsB = float(tA.sum()), float(tB.sum())
        mag = float(tA.abs().sum() + tB.abs().sum() + dly.abs().sum())
        assert abs(lhsA - rhs) <= 2e-2 * mag, (a, "dA", lhsA, rhs, mag)
        assert abs(lhsB - rhs) <= 2e-2 * mag, (a, "dB", lhsB, rhs, mag)


@pytest.mark.parametrize("proj", ["q", "k", "o", "up", "down"])
def test_full_c4_backward_sampled(proj):
    """C4 forward + backward of one projection at full size: Y / dX on sampled rows and dA / dB of
    every fine-tune adapter (over all their rows) against the oracle, plus the Euler identities."""
    batch, w, X, dY = _full(4, proj)
    res = run_smlm(batch, w, X, dY)
    rows = synth.sample_rows(batch, every=131)
    Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, rows=rows)
    dXr, dAr, dBr = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, rows=rows)
    assert parity_err(res.Y.double().numpy()[rows], Y[rows]) <= BF16_TOL
    ft = np.intersect1d(batch.ft_rows(), rows)
    assert parity_err(res.dX.double().numpy()[ft], dXr[ft]) <= BF16_TOL
    for a in sorted(set(batch.row_slot()[batch.ft_rows()].tolist())):
        assert parity_err(res.dA[a], dAr[a]) <= BF16_TOL, (proj, a, "dA")
        assert parity_err(res.dB[a], dBr[a]) <= BF16_TOL, (proj, a, "dB")
    _euler(batch, w, X, dY, res.Y, res.dX, res.dA, res.dB)


def _pools_multi(ws_, r, U, dev):
    from paper_2511_00101_b200 import smlm as S
    pools, keep = [], []
    for w in ws_:
        pool = S.Pool(w.W.shape[1], w.W.shape[0], r, U)
        for a in range(U):
            A, B = w.A[a].to(dev).contiguous(), w.B[a].to(dev).contiguous()
            keep += [A, B]
            assert pool.register(A, B, w.slot_scale[a]) == a
        pools.append(pool)
    return pools, keep


def test_full_c4_gate_up_multi_sampled():
    """C4 gate/up through smlm_forward_multi (shared pre-shrink over X, N = 14336 each)."""
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    batch = synth.config_batch(4)
    ws_ = [synth.config_weights(4, p) for p in ("gate", "up")]
    X, _ = synth.config_activations(4, "gate", batch.S)
    pools, keep = _pools_multi(ws_, 16, 64, dev)
    b = S.Batch.from_synth(batch)
    Ys = [torch.empty(batch.S, 14336, dtype=torch.bfloat16, device=dev) for _ in ws_]
    Vs = [torch.zeros(batch.S, 16, dtype=torch.bfloat16, device=dev) for _ in ws_]
    ws = torch.empty(S.smlm_workspace_size_multi([p.h for p in pools], b) + 256, dtype=torch.uint8, device=dev)
    S.smlm_forward_multi([p.h for p in pools], b, X.to(dev), [w.W.to(dev) for w in ws_], Ys, Vs, ws)
    torch.cuda.synchronize()
    rows = synth.sample_rows(batch, every=151)
    ft = batch.ft_rows()
    ft = ft[batch.row_slot()[ft] >= 0]
    for i, w in enumerate(ws_):
        Y, V = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, rows=rows)
        assert parity_err(Ys[i].double().cpu().numpy()[rows], Y[rows]) <= BF16_TOL, i
        fr = np.intersect1d(ft, rows)
        assert parity_err(Vs[i].double().cpu().numpy()[fr], V[fr]) <= BF16_TOL, i
    for p in pools:
        p.close()


def test_full_c2_qkv_fused_decode_and_o():
    """C2 at full size: 256 decode rows over 32 adapters (r = 16, in = 4096): q/k/v in ONE decode
    launch (smlm_forward_multi) and o alone -- every row against the oracle."""
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", 0)
    batch = synth.config_batch(2)
    ws_ = [synth.config_weights(2, p) for p in ("q", "k", "v", "o")]
    X, _ = synth.config_activations(2, "q", batch.S)
    Xo, _ = synth.config_activations(2, "o", batch.S)
    pools, keep = _pools_multi(ws_, 16, 32, dev)
    b = S.Batch.from_synth(batch)
    Ys = [torch.empty(batch.S, w.W.shape[0], dtype=torch.bfloat16, device=dev) for w in ws_]
    hs = [p.h for p in pools[:3]]
    ws = torch.empty(max(S.smlm_workspace_size_multi(hs, b), S.smlm_workspace_size(pools[3].h, b, False)) + 256,
                     dtype=torch.uint8, device=dev)
    n0 = S.smlm_launch_count()
    S.smlm_forward_multi(hs, b, X.to(dev), [w.W.to(dev) for w in ws_[:3]], Ys[:3], None, ws)
    torch.cuda.synchronize()
    assert S.smlm_launch_count() - n0 == 1, "q/k/v of a decode batch must be ONE launch"
    S.smlm_forward(pools[3].h, b, Xo.to(dev), ws_[3].W.to(dev), Ys[3], None, ws)
    torch.cuda.synchronize()
    for i, w in enumerate(ws_):
        Xi = Xo if i == 3 else X
        Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, Xi)
        assert parity_err(Ys[i].double().cpu().numpy(), Y) <= BF16_TOL, i
    for p in pools:
        p.close()


def test_bench_step_schedule_parity():
    """The exact step bench.py times (C4 workload, forward of the 7 projections of every layer
    through smlm_forward_multi / smlm_forward, backward of every layer in reverse alternating
    two streams, grads into the per-layer flat bucket) -- layer 0's outputs and the LAST layer's
    gradients against the oracle on sampled rows (the workload's own device-generated weights
    and activations, copied to the host)."""
    import bench
    dev = torch.device("cuda", 0)
    wl = bench.Workload(4, 0, dev)
    st = torch.cuda.current_stream(dev)
    wl.step(st)
    torch.cuda.synchronize()
    batch = wl.batch
    rows = synth.sample_rows(batch, every=211)
    ft = batch.ft_rows()
    rs = batch.row_slot()
    for p in synth.PROJECTIONS:
        # forward runs layers 0..7 in order (Y holds layer 7's output); backward runs 7..0 (dX
        # holds layer 0's; every layer has its own gradient bucket and V_save): check Y against
        # layer 7, dX against layer 0, and the gradients of layers 0 and 7
        for Lidx, what in ((bench.N_LAYERS - 1, "fwd"), (0, "bwd"), (bench.N_LAYERS - 1, "grad")):
            e = wl.layers[Lidx][p]
            U = e["A"].shape[0]
            w = synth.Weights(e["W"].cpu(), [e["A"][a].cpu() for a in range(U)], [e["B"][a].cpu() for a in range(U)],
                              [2.0] * U)
            X = wl.X[bench.GROUP_OF[p]].cpu()
            if what == "fwd":
                Y, _ = oracle.forward(batch, w.W, w.A, w.B, w.slot_scale, X, rows=rows)
                assert parity_err(wl.Y[p].double().cpu().numpy()[rows], Y[rows]) <= BF16_TOL, (p, "Y")
            else:
                dY = wl.dY[p].cpu()
                dXr, dAr, dBr = oracle.backward(batch, w.W, w.A, w.B, w.slot_scale, X, dY, rows=rows)
                fr = np.intersect1d(ft, rows)
                if what == "bwd":
                    assert parity_err(wl.dX[p].double().cpu().numpy()[fr], dXr[fr]) <= BF16_TOL, (p, "dX")
                gb = e["grad"]
                for i, s in enumerate(bench.FT_SLOTS):
                    if np.any(rs[ft] == s):
                        assert parity_err(gb.dA(i), dAr[s]) <= BF16_TOL, (p, s, "dA")
                        assert parity_err(gb.dB(i), dBr[s]) <= BF16_TOL, (p, s, "dB")
