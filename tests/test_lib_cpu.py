"""Host-only checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/smlm.h declares, its host planner agrees bit-exactly with the independent Python plan
oracle (oracle/plan.py), and validation errors are reported before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import plan as plan_oracle
from synth import DECODE, EVAL, FINETUNE, PREFILL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def smlm():
    from paper_2511_00101_b200 import build
    build.build()
    import paper_2511_00101_b200.smlm as m
    return m


def header_symbols():
    with open(os.path.join(ROOT, "include", "smlm.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"SMLM_API\s+[\w\s\*]*?\b(smlm_\w+)\s*\(", txt)))


def test_exports_every_header_symbol(smlm):
    syms = header_symbols()
    assert len(syms) >= 16
    lib = ctypes.CDLL(smlm.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(smlm.EXPORTED) == syms


def test_no_gpu_no_fallback(smlm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(smlm.SmlmError) as e:
        smlm.smlm_pool_create(0, 64, 64, 16, 4, smlm.SMLM_BF16)
    assert e.value.code == smlm.SMLM_E_UNSUPPORTED


def _random_batch(rng, cap):
    G = int(rng.integers(1, 50))
    lens = rng.choice([0, 1, 2, 3, 7, 63, 64, 65, 127, 128, 129, 255, 256, 300, 1000], size=G).tolist()
    slots = rng.integers(-1, cap, size=G).tolist()
    modes = rng.integers(0, 4, size=G).tolist()
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    return off, slots, modes


@pytest.mark.parametrize("seed", range(25))
def test_planner_bit_exact_vs_oracle(smlm, seed):
    rng = np.random.default_rng(100 + seed)
    cap = 8
    off, slots, modes = _random_batch(rng, cap)
    reg = np.ones(cap, np.uint8)
    b = smlm.Batch(off, slots, modes)
    for l_long in (1, 16, 64, 129):
        got = smlm.smlm_plan(b, cap, reg, l_long=l_long, backward=False)
        want = plan_oracle.forward_plan(off, slots, modes, l_long=l_long)
        assert got == want
    got = smlm.smlm_plan(b, cap, reg, l_long=64, backward=True)
    assert got == plan_oracle.backward_plan(off, slots, modes)


def test_planner_configs(smlm):
    import synth
    for k in (2, 3, 4, 5):
        for unsorted in (False, True):
            bt = synth.config_batch(k, rank=1, unsorted_decode=unsorted)
            cap = synth.CONFIGS[k].n_adapters
            b = smlm.Batch.from_synth(bt)
            reg = np.ones(cap, np.uint8)
            assert smlm.smlm_plan(b, cap, reg) == plan_oracle.forward_plan(bt.offsets, bt.slots, bt.modes)
            assert smlm.smlm_plan(b, cap, reg, backward=True) == \
                plan_oracle.backward_plan(bt.offsets, bt.slots, bt.modes)


def test_validation_errors(smlm):
    reg = np.array([1, 1, 0, 1], np.uint8)

    def code(off, slots, modes, scale=None):
        try:
            smlm.smlm_plan(smlm.Batch(off, slots, modes, scale), 4, reg)
            return smlm.SMLM_OK
        except smlm.SmlmError as e:
            return e.code
    assert code([0, 3, 5], [0, 1], [0, 3]) == smlm.SMLM_OK
    assert code([1, 3, 5], [0, 1], [0, 3]) == smlm.SMLM_E_INVALID      # off[0] != 0
    assert code([0, 4, 3], [0, 1], [0, 3]) == smlm.SMLM_E_INVALID      # decreasing
    assert code([0, 3, 5], [0, 1], [0, 4]) == smlm.SMLM_E_INVALID      # mode out of range
    assert code([0, 3, 5], [0, 2], [0, 3]) == smlm.SMLM_E_SLOT         # slot not registered
    assert code([0, 3, 5], [0, 7], [0, 3]) == smlm.SMLM_E_SLOT         # slot out of range
    assert code([0, 3, 5], [0, -2], [0, 3]) == smlm.SMLM_E_SLOT
    assert code([0, 3, 5], [0, 1], [0, 3], [1.0, 0.0]) == smlm.SMLM_E_INVALID   # scale 0 rejected
    assert code([0, 3, 5], [0, 1], [0, 3], [1.0, float("nan")]) == smlm.SMLM_E_INVALID
    assert code([0, 0, 0], [0, 1], [0, 3]) == smlm.SMLM_OK              # empty segments
    assert smlm.smlm_plan(smlm.Batch([0], [], []), 4, reg) == []       # G = 0, S = 0
