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


class PeerReduce:
    """Fused cross-rank reduction of the fine-tune gradients (include/smlm.h
    "Fused cross-rank reduction"): instead of an NCCL all-reduce after the backward, every rank's
    dA/dB contraction kernel stores each gradient value into ITS slot of every peer's staging
    buffer over NVLink (peer memory mapped with CUDA IPC) while it runs, signals completion with a
    system-scope counter, and the AdamW step sums the N slots in rank order (deterministic,
    bit-identical replicas) as it updates the parameters.

    Layout (one allocation per rank): stage [2 step parities][N slots][stride] fp32, then the
    int32 ready counter.  Pure plumbing: the reduction arithmetic runs in kernels_opt.cu."""

    def __init__(self, dist, n: int, device):
        from . import smlm as S
        self.S = S
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        N = self.world
        self.n = int(n)
        self.stride = (self.n + 3) // 4 * 4
        self.device = torch.device(device)
        tot = 2 * N * self.stride
        self.buf = torch.zeros(tot + 64, dtype=torch.float32, device=self.device)
        self.stage = self.buf[:tot].view(2, N, self.stride)
        self.ready = self.buf[tot:tot + 1].view(torch.int32)
        h, off = S.smlm_ipc_get_handle(self.buf)
        allh = [None] * N
        dist.all_gather_object(allh, (h, off))
        self.bases = []
        self._opened = []
        for q, (hq, oq) in enumerate(allh):
            if q == self.rank:
                self.bases.append(self.buf.data_ptr())
            else:
                b = S.smlm_ipc_open_handle(hq)
                self._opened.append(b)
                self.bases.append(b + oq)
        own = self.buf.data_ptr()
        # every gradient value written at p (own slot, own buffer) also goes to p + delta[q]
        self.deltas = [self.bases[q] - own for q in range(N) if q != self.rank]
        self.ready_ptrs = [self.bases[q] + 4 * tot for q in range(N)]
        self.steps = 0

    def slot(self, parity: int) -> torch.Tensor:
        """This rank's gradient slot of the given step parity ([n] fp32): bind dA/dB views here."""
        return self.stage[parity, self.rank, :self.n]

    def set_fanout(self, pools):
        for pool in pools:
            self.S.smlm_pool_set_grad_fanout(pool.h if hasattr(pool, "h") else pool, self.deltas)

    def signal(self, stream=None):
        """After this rank's backward of the step (stream order): count it in on every rank."""
        self.S.smlm_fanout_signal(self.ready_ptrs, stream, self.device)
        self.steps += 1

    def ready_target(self) -> int:
        return self.world * self.steps

    def wait(self, stream=None):
        """The stream waits until every rank's slots of the last signalled step are here."""
        self.S.smlm_fanout_wait(self.ready, self.ready_target(), stream)

    def close(self):
        for b in self._opened:
            self.S.smlm_ipc_close_handle(b)
        self._opened = []
