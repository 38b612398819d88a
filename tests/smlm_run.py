"""Test helper: run the CUDA path (through the C ABI binding) on synth inputs."""
from dataclasses import dataclass
from typing import Optional

import torch


@dataclass
class GpuResult:
    Y: torch.Tensor
    V: Optional[torch.Tensor]
    dX: Optional[torch.Tensor]
    dA: torch.Tensor
    dB: torch.Tensor
    plan_fwd: list
    plan_bwd: list


def run_smlm(batch, w, X, dY, dtype=None, backward=True, w_null=False, vsave=True, want_dx=True,
             grads=None, l_long=None, accumulate=False, dA0=None, dB0=None, base_in=None, device=0,
             options=None, dropout=None):
    """dropout: (p, seed) -- LoRA dropout of the fine-tune rows (smlm_batch.dropout_p / _seed)."""
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", device)
    tdt = X.dtype
    dt = S.SMLM_FP32 if tdt == torch.float32 else S.SMLM_BF16
    in_f, out_f = w.W.shape[1], w.W.shape[0]
    ranks = [a.shape[0] for a in w.A]
    r = max(ranks) if ranks else 1          # heterogeneous ranks (f2): the pool takes the largest
    U = len(w.A)
    hetero = any(ra != r for ra in ranks)
    pool = S.Pool(in_f, out_f, r, max(U, 1), dt, device)
    if l_long is not None:
        pool.set_option(S.SMLM_OPT_L_LONG, l_long)
    for opt, val in (options or {}).items():
        pool.set_option(opt, val)
    A = [a.to(dev).contiguous() for a in w.A]
    B = [b.to(dev).contiguous() for b in w.B]
    slots = [pool.register(A[i], B[i], w.slot_scale[i]) for i in range(U)]
    assert slots == list(range(U))
    dA = torch.zeros(max(U, 1), r, in_f, dtype=torch.float32, device=dev) if dA0 is None else dA0.to(dev).clone()
    dB = torch.zeros(max(U, 1), out_f, r, dtype=torch.float32, device=dev) if dB0 is None else dB0.to(dev).clone()
    guards = []
    if hetero:
        # each adapter's gradients in buffers of its own rank, followed by sentinel guards that
        # must survive (no write past [r_a, in] / [out, r_a])
        gA, gB = [], []
        for i in range(U):
            ra = ranks[i]
            bufA = torch.full((ra * in_f + 256,), 12345.0, device=dev)
            bufB = torch.full((out_f * ra + 256,), 12345.0, device=dev)
            bufA[:ra * in_f].copy_(dA[i, :ra].reshape(-1))
            bufB[:out_f * ra].copy_(dB[i, :, :ra].reshape(-1))
            gA.append(bufA)
            gB.append(bufB)
        guards = (gA, gB)
    for i in range(U):
        if grads is None or grads[i]:
            if hetero:
                ra = ranks[i]
                pool.set_grad(i, guards[0][i][:ra * in_f].view(ra, in_f), guards[1][i][:out_f * ra].view(out_f, ra))
            else:
                pool.set_grad(i, dA[i], dB[i])
    b = S.Batch.from_synth(batch) if dropout is None else S.Batch.from_synth(batch, dropout[0], dropout[1])
    Xd = X.to(dev).contiguous()
    Wd = w.W.to(dev).contiguous()
    if w_null:
        Y = base_in.to(dev).clone()
    else:
        Y = torch.full((batch.S, out_f), float("nan"), dtype=tdt, device=dev)
    V = torch.zeros(batch.S, r, dtype=tdt, device=dev) if vsave else None
    pool.forward(b, Xd, None if w_null else Wd, Y, V)
    dX = None
    if backward:
        dX = torch.zeros(batch.S, in_f, dtype=tdt, device=dev) if want_dx else None
        pool.backward(b, Xd, Wd, dY.to(dev).contiguous(), V, dX, accumulate)
    torch.cuda.synchronize()
    if hetero:
        for i in range(U):
            ra = ranks[i]
            gA, gB = guards[0][i], guards[1][i]
            assert bool((gA[ra * in_f:] == 12345.0).all()) and bool((gB[out_f * ra:] == 12345.0).all()), \
                f"adapter {i} (rank {ra}): gradient written past its own rank"
            dA[i].zero_()
            dB[i].zero_()
            dA[i, :ra].copy_(gA[:ra * in_f].view(ra, in_f))
            dB[i, :, :ra].copy_(gB[:out_f * ra].view(out_f, ra))
    res = GpuResult(Y.cpu(), None if V is None else V.cpu(), None if dX is None else dX.cpu(),
                    dA.cpu(), dB.cpu(), pool.plan(b, False), pool.plan(b, True))
    pool.close()
    return res
