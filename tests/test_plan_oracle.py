"""Pins of the Python plan oracle (oracle/plan.py) against a hand-written plan and brute-force
coverage properties."""
import numpy as np
import pytest

from oracle import plan
from synth import DECODE, EVAL, FINETUNE, PREFILL


def test_hand_written_plan():
    # segments: FT 200 rows slot 3 | DECODE 1 slot 5 | DECODE 2 slot 1 | empty | PREFILL 64 slot -1
    #           | DECODE 1 slot 5 | EVAL 10 slot 1
    lens = [200, 1, 2, 0, 64, 1, 10]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    slots = [3, 5, 1, 7, -1, 5, 1]
    modes = [FINETUNE, DECODE, DECODE, DECODE, PREFILL, DECODE, EVAL]
    f = plan.forward_plan(off, slots, modes, l_long=64)
    assert f == [
        [0, 0, 0, 128, 3, FINETUNE],
        [0, 0, 128, 72, 3, FINETUNE],
        [0, 4, 203, 64, -1, PREFILL],
        [1, 0, 200, 3, 2, 0],          # rows 200..202: slots 5, 1, 1
        [2, 0, 0, 1, 2, 0],
        [2, 0, 1, 5, 1, 0],
        [1, 1, 267, 11, 2, 0],         # rows 267..277: slot 5 x1, slot 1 x10
        [2, 1, 0, 1, 10, 0],
        [2, 1, 1, 5, 1, 0],
    ]
    b = plan.backward_plan(off, slots, modes)
    assert b == [[3, 3, 0, 0, 128, 0], [3, 3, 0, 128, 72, 0], [4, 3, 200, 2, 0, 0]]


@pytest.mark.parametrize("seed", range(8))
def test_coverage_properties(seed):
    rng = np.random.default_rng(seed)
    G = int(rng.integers(1, 40))
    lens = rng.choice([0, 1, 2, 5, 63, 64, 65, 127, 128, 129, 300], size=G).tolist()
    slots = rng.integers(-1, 6, size=G).tolist()
    modes = rng.integers(0, 4, size=G).tolist()
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    S = int(off[-1])
    L = int(rng.choice([1, 16, 64, 200]))
    f = plan.forward_plan(off, slots, modes, l_long=L)
    cover = np.zeros(S, int)
    seg_of = np.repeat(np.arange(G), lens)
    tiles = {}
    for rec in f:
        if rec[0] == 0:
            _, g, r0, n, s, m = rec
            assert 1 <= n <= 128 and lens[g] >= L
            assert off[g] <= r0 and r0 + n <= off[g + 1] and (r0 - off[g]) % 128 == 0
            assert s == slots[g] and m == modes[g]
            cover[r0:r0 + n] += 1
        elif rec[0] == 1:
            _, t, r0, n, nb, _ = rec
            assert 1 <= n <= 128
            assert all(0 < lens[seg_of[x]] < L for x in range(r0, r0 + n))
            cover[r0:r0 + n] += 1
            tiles[t] = (r0, n, nb, [])
        elif rec[0] == 2:
            _, t, b, s, cnt, _ = rec
            tiles[t][3].append((b, s, cnt))
    assert np.all(cover == 1)
    for t, (r0, n, nb, blks) in tiles.items():
        assert [b for b, _, _ in blks] == list(range(nb))
        ss = [s for _, s, _ in blks]
        assert ss == sorted(set(ss)) and all(s >= 0 for s in ss)
        row_slots = [slots[seg_of[x]] for x in range(r0, r0 + n)]
        for _, s, cnt in blks:
            assert cnt == row_slots.count(s)
        assert sum(c for _, _, c in blks) == sum(1 for s in row_slots if s >= 0)
    b = plan.backward_plan(off, slots, modes)
    bc = np.zeros(S, int)
    prev = None
    for rec in b:
        if rec[0] == 3:
            _, s, g, r0, n, _ = rec
            assert modes[g] == FINETUNE and slots[g] == s
            key = (s, g, r0)
            assert prev is None or key > prev
            prev = key
            bc[r0:r0 + n] += 1
    ft = np.array([modes[seg_of[x]] == FINETUNE for x in range(S)], bool)
    assert np.array_equal(bc, ft.astype(int))
