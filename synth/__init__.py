"""Seeded synthetic inputs for SMLM (shared by the oracle side and the CUDA side).

This module holds NO arithmetic of the method: it only draws random numbers and
lays out batch structure (segment offsets, adapter slots, modes, scales).  Both the
oracle tests and the CUDA path read the exact same tensors from here; neither
side imports the other.

Recipe (SURVEY.md §8(d) "Synthetic inputs"; BASELINE.json `configs`):
  * distributions: X ~ N(0,1); W ~ N(0,1/in); A ~ N(0,1/in); B ~ N(0,1/(16 r)); dY ~ N(0,1)
    (B != 0 on purpose: the paper's gaussian init sets B=0 at step 0, Table 5,
    which would make dA trivially zero).
  * slot scale s = alpha/r with alpha = 2r  =>  s = 2   (Table 5: r=8, alpha=16).
  * C1: one CPU torch.Generator seeded 1001, draws W, A_0..A_{U-1}, B_0..B_{U-1}, X, dY (fp32).
  * C2..C5 weights: generator seed 1000+10k+p (k = config number, p = projection index
    q,k,v,o,gate,up,down = 0..6): W, all A, all B.  Rank independent (adapters replicated).
  * C2..C5 inputs: seed 5000+10k+p+7919*rank: X then dY.
  * C2..C5 batch structure: seed 9000+k+7919*rank: prefill lengths, then slot draws.
  * Row order F, E, P, D (fine-tune, eval, prefill, decode), Alg. 1.
  * Values are cast to bf16 AFTER scaling (C1 stays fp32).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

FINETUNE, EVAL, PREFILL, DECODE = 0, 1, 2, 3
MODE_NAMES = {FINETUNE: "finetune", EVAL: "eval", PREFILL: "prefill", DECODE: "decode"}

# Llama-3-8B projection shapes (in, out); GQA k/v out = 1024 (App. E).
PROJECTIONS = ["q", "k", "v", "o", "gate", "up", "down"]
PROJ_SHAPES = {
    "q": (4096, 4096), "k": (4096, 1024), "v": (4096, 1024), "o": (4096, 4096),
    "gate": (4096, 14336), "up": (4096, 14336), "down": (14336, 4096),
}


@dataclass
class Batch:
    """A segmented mixed batch (Alg. 1 Require)."""
    offsets: np.ndarray          # int32 [G+1]
    slots: np.ndarray            # int32 [G]   (-1 = base only)
    modes: np.ndarray            # int8  [G]
    seg_scale: Optional[np.ndarray] = None   # float32 [G] or None (= 1)

    @property
    def S(self) -> int:
        return int(self.offsets[-1])

    @property
    def G(self) -> int:
        return int(len(self.slots))

    def row_slot(self) -> np.ndarray:
        out = np.full(self.S, -1, np.int32)
        for g in range(self.G):
            out[self.offsets[g]:self.offsets[g + 1]] = self.slots[g]
        return out

    def row_mode(self) -> np.ndarray:
        out = np.zeros(self.S, np.int8)
        for g in range(self.G):
            out[self.offsets[g]:self.offsets[g + 1]] = self.modes[g]
        return out

    def ft_rows(self) -> np.ndarray:
        return np.nonzero(self.row_mode() == FINETUNE)[0].astype(np.int64)


@dataclass
class Weights:
    """Base weight plus an adapter pool for one (layer, projection)."""
    W: torch.Tensor                  # [out, in]
    A: List[torch.Tensor]            # U x [r, in]
    B: List[torch.Tensor]            # U x [out, r]
    slot_scale: List[float] = field(default_factory=list)

    @property
    def in_features(self) -> int:
        return self.W.shape[1]

    @property
    def out_features(self) -> int:
        return self.W.shape[0]

    @property
    def rank(self) -> int:
        return self.A[0].shape[0] if self.A else 0


def batch_from_lengths(lengths: Sequence[int], slots: Sequence[int], modes: Sequence[int],
                       seg_scale: Optional[Sequence[float]] = None) -> Batch:
    off = np.zeros(len(lengths) + 1, np.int32)
    off[1:] = np.cumsum(np.asarray(lengths, np.int64))
    return Batch(off, np.asarray(slots, np.int32), np.asarray(modes, np.int8),
                 None if seg_scale is None else np.asarray(seg_scale, np.float32))


def draw_weights(gen: torch.Generator, in_f: int, out_f: int, r: int, n_adapters: int,
                 dtype=torch.bfloat16, slot_scale: float = 2.0) -> Weights:
    W = torch.randn(out_f, in_f, generator=gen) / math.sqrt(in_f)
    A = [torch.randn(r, in_f, generator=gen) / math.sqrt(in_f) for _ in range(n_adapters)]
    B = [torch.randn(out_f, r, generator=gen) / (4.0 * math.sqrt(r)) for _ in range(n_adapters)]
    return Weights(W.to(dtype), [a.to(dtype) for a in A], [b.to(dtype) for b in B],
                   [float(slot_scale)] * n_adapters)


def draw_activations(gen: torch.Generator, S: int, in_f: int, out_f: int, dtype=torch.bfloat16):
    X = torch.randn(S, in_f, generator=gen).to(dtype)
    dY = torch.randn(S, out_f, generator=gen).to(dtype)
    return X, dY


# ----------------------------------------------------------------------------------------
# C1: tiny fp32 case (SURVEY.md §8(c) pin 9, §8(d) C1)
# ----------------------------------------------------------------------------------------
C1_IN = C1_OUT = 64
C1_RANK = 4


def c1_batch() -> Batch:
    return batch_from_lengths([12, 8, 8, 4], [0, 1, 2, 0], [FINETUNE, EVAL, PREFILL, DECODE],
                              [1.0, 0.5, 1.0, 2.0])


def c1_inputs():
    """Returns (batch, weights, X, dY), all fp32, drawn in the SURVEY order from seed 1001."""
    g = torch.Generator().manual_seed(1001)
    w = draw_weights(g, C1_IN, C1_OUT, C1_RANK, 3, dtype=torch.float32, slot_scale=2.0)
    batch = c1_batch()
    X, dY = draw_activations(g, batch.S, C1_IN, C1_OUT, dtype=torch.float32)
    return batch, w, X, dY


# ----------------------------------------------------------------------------------------
# C2..C5 (BASELINE.json configs[1..4])
# ----------------------------------------------------------------------------------------
@dataclass
class ConfigSpec:
    k: int                      # config number (2..5)
    name: str
    projections: List[str]
    rank: int
    n_adapters: int


CONFIGS = {
    2: ConfigSpec(2, "C2-decode", ["q", "k", "v", "o"], 16, 32),
    3: ConfigSpec(3, "C3-prefill", ["gate", "up", "down"], 64, 8),
    4: ConfigSpec(4, "C4-unified", PROJECTIONS, 16, 64),
    5: ConfigSpec(5, "C5-dp", PROJECTIONS, 16, 256),
}


def _group_by_slot(slots: np.ndarray, mode: int):
    """Decode rows grouped by slot: one segment per distinct slot, ascending."""
    uniq, counts = np.unique(slots, return_counts=True)
    return list(counts), list(uniq), [mode] * len(uniq)


def config_batch(k: int, rank: int = 0, unsorted_decode: bool = False) -> Batch:
    """Batch structure for config k on a given DP rank (seed 9000 + k + 7919*rank)."""
    spec = CONFIGS[k]
    g = torch.Generator().manual_seed(9000 + k + 7919 * rank)
    lengths, slots, modes = [], [], []
    if k == 2:
        s = torch.randint(0, spec.n_adapters, (256,), generator=g).numpy().astype(np.int32)
        if unsorted_decode:
            lengths, slots, modes = [1] * 256, list(s), [DECODE] * 256
        else:
            lengths, slots, modes = _group_by_slot(s, DECODE)
    elif k == 3:
        pl = torch.randint(512, 2049, (8,), generator=g).tolist()
        ps = torch.randperm(8, generator=g).tolist()
        lengths, slots, modes = pl, ps, [PREFILL] * 8
    elif k in (4, 5):
        pl = torch.randint(512, 2049, (8,), generator=g).tolist()
        ps = torch.randint(0, spec.n_adapters, (8,), generator=g).tolist()
        ds = torch.randint(0, spec.n_adapters, (128,), generator=g).numpy().astype(np.int32)
        lengths = [1024] * 4 + pl
        slots = [0, 1, 2, 3] + ps
        modes = [FINETUNE] * 4 + [PREFILL] * 8
        if unsorted_decode:
            lengths += [1] * 128
            slots += list(ds)
            modes += [DECODE] * 128
        else:
            dl, dsl, dm = _group_by_slot(ds, DECODE)
            lengths += dl
            slots += dsl
            modes += dm
    else:
        raise ValueError(k)
    return batch_from_lengths(lengths, slots, modes)


def config_weights(k: int, proj: str, dtype=torch.bfloat16, in_out=None, n_adapters=None) -> Weights:
    spec = CONFIGS[k]
    p = PROJECTIONS.index(proj)
    in_f, out_f = in_out if in_out is not None else PROJ_SHAPES[proj]
    g = torch.Generator().manual_seed(1000 + 10 * k + p)
    return draw_weights(g, in_f, out_f, spec.rank, n_adapters or spec.n_adapters, dtype=dtype)


def config_activations(k: int, proj: str, S: int, rank: int = 0, dtype=torch.bfloat16, in_out=None):
    p = PROJECTIONS.index(proj)
    in_f, out_f = in_out if in_out is not None else PROJ_SHAPES[proj]
    g = torch.Generator().manual_seed(5000 + 10 * k + p + 7919 * rank)
    return draw_activations(g, S, in_f, out_f, dtype=dtype)


def random_case(seed: int, in_f: int, out_f: int, r: int, n_adapters: int, lengths: Sequence[int],
                modes: Sequence[int], slots: Optional[Sequence[int]] = None,
                seg_scale: Optional[Sequence[float]] = None, dtype=torch.bfloat16,
                slot_scale: float = 2.0):
    """Small generic case for parity tests: returns (batch, weights, X, dY)."""
    g = torch.Generator().manual_seed(seed)
    w = draw_weights(g, in_f, out_f, r, n_adapters, dtype=dtype, slot_scale=slot_scale)
    if slots is None:
        slots = torch.randint(-1, n_adapters, (len(lengths),), generator=g).tolist()
    batch = batch_from_lengths(lengths, slots, modes, seg_scale)
    X, dY = draw_activations(g, batch.S, in_f, out_f, dtype=dtype)
    return batch, w, X, dY


def sample_rows(batch: Batch, every: int = 37) -> np.ndarray:
    """Deterministic row sample: first and last row of each segment plus every `every`-th row
    (SURVEY.md §8(d) "Oracle timing beside it")."""
    rows = set(range(0, batch.S, every))
    for g in range(batch.G):
        a, b = int(batch.offsets[g]), int(batch.offsets[g + 1])
        if b > a:
            rows.add(a)
            rows.add(b - 1)
    return np.array(sorted(rows), np.int64)


def lora_param_count(rank: int, projections: Sequence[str] = tuple(PROJECTIONS)) -> int:
    """Elements of one adapter's A and B over the given Llama-3-8B projections (no arithmetic of the
    method: shapes only)."""
    return sum(rank * PROJ_SHAPES[p][0] + PROJ_SHAPES[p][1] * rank for p in projections)


def draw_adamw_state(seed: int, n: int, step: int = 1):
    """Seeded fp32 AdamW inputs of n elements (CPU tensors): parameters ~ N(0, 0.02) (the
    gaussian LoRA init scale), a gradient sum ~ N(0, 1e-3), and, for step > 1, moments of a run
    in progress (exp_avg ~ N(0, 1e-4), exp_avg_sq ~ |N(0, 1e-6)|)."""
    g = torch.Generator().manual_seed(seed)
    p = torch.randn(n, generator=g) * 0.02
    grad = torch.randn(n, generator=g) * 1e-3
    if step > 1:
        m = torch.randn(n, generator=g) * 1e-4
        v = (torch.randn(n, generator=g) * 1e-6).abs()
    else:
        m = torch.zeros(n)
        v = torch.zeros(n)
    return p, m, v, grad


# ----------------------------------------------------------------------------------------
# LoRA dropout mask (Table 5 lora_dropout 0.05; R13):
# a counter-based generator, so the oracle gets the mask as an explicit input while the CUDA
# path draws the same bits from (seed, row, column) with its own implementation of this hash
# (no shared code: csrc implements it in CUDA).  It is a random-number generator, not method
# arithmetic.
#   thr = round(p * 65536)  (drop probability quantised to 1/65536; keep scale 65536/(65536-thr))
#   element (t, k) of X [S, in]:  c = t * ceil(in/2) + floor(k/2)   (uint32, wrapping)
#     h = lowbias32(lowbias32(c ^ seed_lo) ^ seed_hi)
#     u = (k odd) ? h >> 16 : h & 0xffff ;   kept  <=>  u >= thr
# ----------------------------------------------------------------------------------------
def dropout_threshold(p: float) -> int:
    if not (0.0 <= p < 1.0):
        raise ValueError("dropout p must be in [0, 1)")
    return int(round(p * 65536.0))


def dropout_effective_p(p: float) -> float:
    """The drop probability the threshold realises (what the oracle's keep scale uses)."""
    return dropout_threshold(p) / 65536.0


def _lowbias32(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x = (x * np.uint32(0x7FEB352D)).astype(np.uint32)
    x ^= x >> np.uint32(15)
    x = (x * np.uint32(0x846CA68B)).astype(np.uint32)
    x ^= x >> np.uint32(16)
    return x


def dropout_keep(seed: int, p: float, S: int, in_f: int) -> np.ndarray:
    """bool [S, in_f]: True where the element is kept."""
    thr = dropout_threshold(p)
    seed_lo, seed_hi = np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF)
    half = (in_f + 1) // 2
    t = np.arange(S, dtype=np.uint64)[:, None]
    k = np.arange(in_f, dtype=np.uint64)[None, :]
    c = ((t * np.uint64(half) + k // np.uint64(2)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    with np.errstate(over="ignore"):
        h = _lowbias32(_lowbias32(c ^ seed_lo) ^ seed_hi)
    u = np.where((k % 2).astype(bool), h >> np.uint32(16), h & np.uint32(0xFFFF))
    return u >= np.uint32(thr)
