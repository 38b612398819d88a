"""Flat adapter parameters and the AdamW step after the SMLM backward.

PAPER.md P:420-422: the fine-tune jobs share one backward and each trainer updates only its own
adapter (MixedLoRAModelForTrainer).  Here every trained (pool, slot) adapter lives in ONE flat
layout used by four fp32 buffers (master weights, exp_avg, exp_avg_sq, gradient) and one bf16
buffer (the working copy the pools borrow):

    [ A_0 (r*in) | B_0 (out*r) | A_1 | B_1 | ... ]      each piece padded to 8 elements

so that the SMLM backward writes dA/dB straight into gradient views, the data-parallel
all-reduce is one NCCL call over the flat gradient, and the optimizer is one launch
(`smlm_adamw_step`).  Argument marshalling only: the arithmetic runs in kernels_opt.cu.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch

from . import smlm as S


def _pad8(n: int) -> int:
    return (n + 7) // 8 * 8


class AdapterParams:
    """Flat storage of the trained adapters: shapes = [(rank, in_features, out_features), ...]."""

    def __init__(self, shapes: Sequence[Tuple[int, int, int]], device="cuda"):
        self.shapes = [tuple(int(v) for v in s) for s in shapes]
        self.offsets: List[Tuple[int, int]] = []
        off = 0
        for r, i, o in self.shapes:
            a = off
            off += _pad8(r * i)
            b = off
            off += _pad8(o * r)
            self.offsets.append((a, b))
        self.n = off
        f32 = dict(dtype=torch.float32, device=device)
        self.master = torch.zeros(self.n, **f32)
        self.exp_avg = torch.zeros(self.n, **f32)
        self.exp_avg_sq = torch.zeros(self.n, **f32)
        self.grad = torch.zeros(self.n, **f32)
        self.bf16 = torch.zeros(self.n, dtype=torch.bfloat16, device=device)

    def _view(self, buf, k: int, which: str):
        r, i, o = self.shapes[k]
        a, b = self.offsets[k]
        return buf[a:a + r * i].view(r, i) if which == "A" else buf[b:b + o * r].view(o, r)

    # bf16 working copies (what a pool borrows) and fp32 gradient views (what the backward writes)
    def A(self, k: int) -> torch.Tensor:
        return self._view(self.bf16, k, "A")

    def B(self, k: int) -> torch.Tensor:
        return self._view(self.bf16, k, "B")

    def dA(self, k: int) -> torch.Tensor:
        return self._view(self.grad, k, "A")

    def dB(self, k: int) -> torch.Tensor:
        return self._view(self.grad, k, "B")

    def load(self, k: int, A: torch.Tensor, B: torch.Tensor):
        """Initial values of adapter k (master fp32 and the bf16 working copy)."""
        self._view(self.master, k, "A").copy_(A)
        self._view(self.master, k, "B").copy_(B)
        self.A(k).copy_(self._view(self.master, k, "A"))
        self.B(k).copy_(self._view(self.master, k, "B"))


class AdamW:
    """AdamW over an AdapterParams store.  Defaults: PAPER.md Table 5 lr 2e-5; the HF Trainer
    optimizer defaults otherwise (R9): betas (0.9, 0.999), eps 1e-8, weight_decay 0,
    max_grad_norm 1.0."""

    def __init__(self, params: AdapterParams, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, max_grad_norm: float = 1.0):
        self.p = params
        self.lr, self.betas, self.eps, self.wd, self.max_norm = lr, tuple(betas), eps, weight_decay, max_grad_norm
        self.t = 0
        nws = S.smlm_adamw_workspace_size() // 4
        self.ws = torch.empty(max(nws, 1), dtype=torch.float32, device=params.master.device)

    def step(self, grad_scale: float = 1.0, zero_grad: bool = True, lr: float = None, stream=None):
        """One step on the accumulated gradient (grad_scale: e.g. 1/(world * accumulation))."""
        self.t += 1
        S.smlm_adamw_step(self.p.master, self.p.exp_avg, self.p.exp_avg_sq, self.p.grad, self.p.bf16, self.t,
                          self.lr if lr is None else lr, self.betas[0], self.betas[1], self.eps, self.wd,
                          grad_scale, self.max_norm, zero_grad, self.ws, stream)
