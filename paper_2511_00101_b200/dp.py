"""Data-parallel plumbing for SMLM (BASELINE.json north_star).

Request batches are independent per GPU; base weights and adapters are replicated; the only
exchange is a SUM all-reduce of the fine-tune adapters' fp32 dA/dB (PAPER.md P:422 masking: only
fine-tune adapters carry gradients).  A flat bucket holds the dA/dB of the fine-tune slots so
that a single NCCL call reduces them (bench.py: one bucket per layer whose per-projection
GradBucket views share one buffer); on CUDA the call is issued on a side stream that waits on an
event recorded after the layer's backward, so it overlaps the next layer's backward.  Pure
plumbing: no SMLM arithmetic lives here.
"""
from __future__ import annotations

from typing import Sequence

import torch


class GradBucket:
    """Flat fp32 buffer [ |slots| * r*in  |  |slots| * out*r ] with per-slot dA/dB views."""

    def __init__(self, slots: Sequence[int], r: int, in_f: int, out_f: int, device="cpu", flat=None):
        """flat: an existing fp32 buffer of numel() elements to use (e.g. a slice of a per-layer bucket)."""
        self.slots = list(slots)
        self.r, self.in_f, self.out_f = r, in_f, out_f
        self.nA, self.nB = r * in_f, out_f * r
        n = len(self.slots) * (self.nA + self.nB)
        if flat is not None and (flat.numel() != n or flat.dtype != torch.float32):
            raise ValueError("GradBucket: flat must be fp32 with len(slots) * r * (in + out) elements")
        self.flat = torch.zeros(n, dtype=torch.float32, device=device) if flat is None else flat

    def dA(self, i: int) -> torch.Tensor:
        return self.flat[i * self.nA:(i + 1) * self.nA].view(self.r, self.in_f)

    def dB(self, i: int) -> torch.Tensor:
        o = len(self.slots) * self.nA
        return self.flat[o + i * self.nB:o + (i + 1) * self.nB].view(self.out_f, self.r)

    def bind(self, pool):
        """Bind the views as the pool's gradient buffers of the fine-tune slots."""
        for i, s in enumerate(self.slots):
            pool.set_grad(s, self.dA(i), self.dB(i))


class AllReduce:
    """SUM all-reduce of gradient buckets; on CUDA overlapped on a side stream."""

    def __init__(self, dist, device):
        self.dist = dist
        self.cuda = torch.device(device).type == "cuda"
        self.stream = torch.cuda.Stream(device) if self.cuda else None

    def __call__(self, bucket, main_stream=None):
        """bucket: a GradBucket, an optim.AdapterParams (its flat gradient) or a flat tensor."""
        flat = bucket if isinstance(bucket, torch.Tensor) else getattr(bucket, "flat", None)
        if flat is None:
            flat = bucket.grad
        if self.dist is None:
            return
        if not self.cuda:
            self.dist.all_reduce(flat, op=self.dist.ReduceOp.SUM)
            return
        main = main_stream or torch.cuda.current_stream(flat.device)
        ev = torch.cuda.Event()
        ev.record(main)
        self.stream.wait_event(ev)
        with torch.cuda.stream(self.stream):
            self.dist.all_reduce(flat, op=self.dist.ReduceOp.SUM)

    def join(self, main_stream=None):
        """Make the main stream wait for every issued all-reduce."""
        if self.cuda and self.dist is not None:
            (main_stream or torch.cuda.current_stream()).wait_stream(self.stream)
