"""Flat adapter parameters and the AdamW step after the SMLM backward.

PAPER.md P:420-422: the fine-tune jobs share one backward and each trainer updates only its own
adapter (MixedLoRAModelForTrainer); every job is an HF Trainer of its own (Table 5),
so gradient clipping, the step count, the learning rate and the accumulation schedule are PER
JOB.  Every trained (pool, slot) adapter lives in ONE flat layout used by four fp32 buffers
(master weights, exp_avg, exp_avg_sq, gradient) and one bf16 buffer (the working copy the pools
borrow); the adapters of one job are contiguous:

    [ job 0: A_0 (r*in) | B_0 (out*r) | ... | job 1: ... ]      each piece padded to 8 elements

so that the SMLM backward writes dA/dB straight into gradient views, the data-parallel
all-reduce is one NCCL call over the flat gradient (the SUM is elementwise, so jobs do not mix),
and each job's optimizer step is one `smlm_adamw_step` over its own sub-range with its own clip
norm and step count.  Argument marshalling only: the arithmetic runs in kernels_opt.cu.
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import torch

from . import smlm as S


def _pad8(n: int) -> int:
    return (n + 7) // 8 * 8


class AdapterParams:
    """Flat storage of the trained adapters: shapes = [(rank, in_features, out_features), ...];
    jobs[k] = the fine-tune job adapter k belongs to (default: one job per adapter).  The adapters
    of a job must be consecutive in `shapes` (one contiguous sub-range per job)."""

    def __init__(self, shapes: Sequence[Tuple[int, int, int]], device="cuda", jobs: Optional[Sequence[int]] = None,
                 grad: Optional[torch.Tensor] = None):
        self.shapes = [tuple(int(v) for v in s) for s in shapes]
        self.jobs = list(range(len(self.shapes))) if jobs is None else [int(j) for j in jobs]
        if len(self.jobs) != len(self.shapes):
            raise ValueError("AdapterParams: one job id per adapter")
        self.offsets: List[Tuple[int, int]] = []
        self.job_range: Dict[int, Tuple[int, int]] = {}
        off = 0
        for k, (r, i, o) in enumerate(self.shapes):
            j = self.jobs[k]
            if j in self.job_range and self.jobs[k - 1] != j:
                raise ValueError("AdapterParams: the adapters of a job must be consecutive")
            a = off
            off += _pad8(r * i)
            b = off
            off += _pad8(o * r)
            self.offsets.append((a, b))
            lo = self.job_range.get(j, (a, a))[0]
            self.job_range[j] = (lo, off)
        self.n = off
        f32 = dict(dtype=torch.float32, device=device)
        self.master = torch.zeros(self.n, **f32)
        self.exp_avg = torch.zeros(self.n, **f32)
        self.exp_avg_sq = torch.zeros(self.n, **f32)
        # the gradient may live elsewhere (dp.PeerReduce: this rank's staging slot)
        self.grad = torch.zeros(self.n, **f32) if grad is None else grad
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

    def job(self, j: int):
        """(master, exp_avg, exp_avg_sq, grad, bf16) views of job j's contiguous sub-range."""
        lo, hi = self.job_range[j]
        return tuple(buf[lo:hi] for buf in (self.master, self.exp_avg, self.exp_avg_sq, self.grad, self.bf16))

    def load(self, k: int, A: torch.Tensor, B: torch.Tensor):
        """Initial values of adapter k (master fp32 and the bf16 working copy)."""
        self._view(self.master, k, "A").copy_(A)
        self._view(self.master, k, "B").copy_(B)
        self.A(k).copy_(self._view(self.master, k, "A"))
        self.B(k).copy_(self._view(self.master, k, "B"))


class AdamW:
    """Per-job AdamW over an AdapterParams store.  Defaults: PAPER.md Table 5 lr 2e-5; the HF
    Trainer optimizer defaults otherwise (R12): betas (0.9, 0.999), eps 1e-8,
    weight_decay 0, max_grad_norm 1.0 -- each job clips by its OWN gradient norm and keeps its own
    step count, so jobs with different accumulation schedules share one store."""

    def __init__(self, params: AdapterParams, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, max_grad_norm: float = 1.0):
        self.p = params
        self.lr, self.betas, self.eps, self.wd, self.max_norm = lr, tuple(betas), eps, weight_decay, max_grad_norm
        self.t: Dict[int, int] = {j: 0 for j in params.job_range}
        nws = S.smlm_adamw_workspace_size() // 4
        self.ws = torch.empty(max(nws, 1), dtype=torch.float32, device=params.master.device)

    def step(self, jobs: Optional[Iterable[int]] = None, grad_scale: float = 1.0, zero_grad: bool = True,
             lr: Optional[float] = None, stream=None, peer=None, parity: int = 0):
        """One step of each listed job (default: all) on its accumulated gradient (grad_scale: e.g.
        1/(world * accumulation)); a job steps when ITS accumulation window closes.
        peer: a dp.PeerReduce -- the gradient is the rank-ordered sum of the peer slots of the given
        step parity (store.grad must be peer.slot(parity)), reduced inside the step."""
        for j in (sorted(self.p.job_range) if jobs is None else jobs):
            self.t[j] += 1
            m, ea, es, g, pb = self.p.job(j)
            lr_j = self.lr if lr is None else lr
            if peer is None:
                S.smlm_adamw_step(m, ea, es, g, pb, self.t[j], lr_j, self.betas[0], self.betas[1], self.eps, self.wd,
                                  grad_scale, self.max_norm, zero_grad, self.ws, stream)
            else:
                lo, hi = self.p.job_range[j]
                S.smlm_adamw_step_reduce(m, ea, es, peer.stage[parity, 0, lo:], peer.world, peer.stride, peer.rank,
                                         pb, hi - lo, self.t[j], lr_j, self.betas[0], self.betas[1], self.eps, self.wd,
                                         grad_scale, self.max_norm, zero_grad, peer.ready, peer.ready_target(),
                                         self.ws, stream)
