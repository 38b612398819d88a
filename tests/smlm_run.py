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
             grads=None, l_long=None, accumulate=False, dA0=None, dB0=None, base_in=None, device=0):
    from paper_2511_00101_b200 import smlm as S
    dev = torch.device("cuda", device)
    tdt = X.dtype
    dt = S.SMLM_FP32 if tdt == torch.float32 else S.SMLM_BF16
    in_f, out_f = w.W.shape[1], w.W.shape[0]
    r = w.A[0].shape[0]
    U = len(w.A)
    pool = S.Pool(in_f, out_f, r, max(U, 1), dt, device)
    if l_long is not None:
        pool.set_option(S.SMLM_OPT_L_LONG, l_long)
    A = [a.to(dev).contiguous() for a in w.A]
    B = [b.to(dev).contiguous() for b in w.B]
    slots = [pool.register(A[i], B[i], w.slot_scale[i]) for i in range(U)]
    assert slots == list(range(U))
    dA = torch.zeros(max(U, 1), r, in_f, dtype=torch.float32, device=dev) if dA0 is None else dA0.to(dev).clone()
    dB = torch.zeros(max(U, 1), out_f, r, dtype=torch.float32, device=dev) if dB0 is None else dB0.to(dev).clone()
    for i in range(U):
        if grads is None or grads[i]:
            pool.set_grad(i, dA[i], dB[i])
    b = S.Batch.from_synth(batch)
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
    res = GpuResult(Y.cpu(), None if V is None else V.cpu(), None if dX is None else dX.cpu(),
                    dA.cpu(), dB.cpu(), pool.plan(b, False), pool.plan(b, True))
    pool.close()
    return res
