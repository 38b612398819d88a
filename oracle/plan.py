"""Canonical SMLM work plan, re-derived independently in Python (TEST INFRASTRUCTURE ONLY).

The plan is the integer bookkeeping of the segment scheduler (the paper's
segment descriptors F/E/P/D and offsets, Alg. 1).  The product planner is
host C++ (paper_2511_00101_b200/csrc/planner.cpp); this file shares no code with it and the two
must agree bit-exactly (tests/test_plan.py).  Rules:

  parameters: TILE_M = 128 rows, L_long (default 64)
  forward records (6 x int32 each), in this order:
    [0, g, row0, rows, slot, mode]  long m-tiles: every segment with len >= L_long, in segment
                                    order, tiles row0 = off[g] + 128 k (k ascending), rows <= 128
    [1, t, row0, rows, nblk, 0]     short tile t: the rows of maximal runs of consecutive short
                                    segments (0 < len < L_long; empty segments do not break a
                                    run, long ones do), chopped into <= 128 consecutive rows;
    [2, t, b, slot, nrows, 0]       followed by its nblk adapter blocks: the distinct slots >= 0
                                    among the tile's rows, ascending, with their row counts
  backward records:
    [3, slot, g, row0, rows, 0]     fine-tune m-tiles (segment aligned, any length > 0), ordered
                                    by slot ascending (-1 first), then segment, then k.  This is
                                    the fixed dA/dB reduction order.
    [4, slot, ft_tokens, n_tiles, 0, 0]  per slot >= 0 with fine-tune rows, ascending
"""
from __future__ import annotations

from typing import List

TILE_M = 128
FINETUNE = 0


def forward_plan(offsets, slots, modes, l_long: int = 64, tile_m: int = TILE_M) -> List[List[int]]:
    G = len(slots)
    lens = [int(offsets[g + 1]) - int(offsets[g]) for g in range(G)]
    recs: List[List[int]] = []
    for g in range(G):
        if lens[g] >= l_long and lens[g] > 0:
            k = 0
            while k * tile_m < lens[g]:
                rows = min(tile_m, lens[g] - k * tile_m)
                recs.append([0, g, int(offsets[g]) + k * tile_m, rows, int(slots[g]), int(modes[g])])
                k += 1
    # short runs
    runs = []  # list of lists of (row, slot)
    cur = []
    for g in range(G):
        if lens[g] == 0:
            continue
        if lens[g] >= l_long:
            if cur:
                runs.append(cur)
                cur = []
            continue
        for t in range(int(offsets[g]), int(offsets[g + 1])):
            cur.append((t, int(slots[g])))
    if cur:
        runs.append(cur)
    tile = 0
    for run in runs:
        for i in range(0, len(run), tile_m):
            chunk = run[i:i + tile_m]
            counts = {}
            for (_, s) in chunk:
                if s >= 0:
                    counts[s] = counts.get(s, 0) + 1
            recs.append([1, tile, chunk[0][0], len(chunk), len(counts), 0])
            for b, s in enumerate(sorted(counts)):
                recs.append([2, tile, b, s, counts[s], 0])
            tile += 1
    return recs


def backward_plan(offsets, slots, modes, tile_m: int = TILE_M) -> List[List[int]]:
    G = len(slots)
    ft = [g for g in range(G) if int(modes[g]) == FINETUNE and int(offsets[g + 1]) > int(offsets[g])]
    recs: List[List[int]] = []
    for s in sorted(set(int(slots[g]) for g in ft)):
        for g in ft:
            if int(slots[g]) != s:
                continue
            n = int(offsets[g + 1]) - int(offsets[g])
            for k in range(0, n, tile_m):
                recs.append([3, s, g, int(offsets[g]) + k, min(tile_m, n - k), 0])
    for s in sorted(set(int(slots[g]) for g in ft if int(slots[g]) >= 0)):
        tok = sum(int(offsets[g + 1]) - int(offsets[g]) for g in ft if int(slots[g]) == s)
        ntl = sum(-(-(int(offsets[g + 1]) - int(offsets[g])) // tile_m) for g in ft if int(slots[g]) == s)
        recs.append([4, s, tok, ntl, 0, 0])
    return recs
