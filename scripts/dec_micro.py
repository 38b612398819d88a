"""Decode-path micro-benchmark: per-kernel device time (library CUDA events) for C2 projections,
back-to-back calls over 8 rotated weight sets."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

k = int(os.environ.get("CFG", "2"))
spec = synth.CONFIGS[k]
batch = synth.config_batch(k)
b = S.Batch.from_synth(batch)
dev = torch.device("cuda", 0)
for proj in spec.projections:
    in_f, out_f = synth.PROJ_SHAPES[proj]
    X = torch.randn(batch.S, in_f, device=dev).to(torch.bfloat16)
    Y = torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev)
    sets = []
    for _ in range(8):
        W = (torch.randn(out_f, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
        A = (torch.randn(spec.n_adapters, spec.rank, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
        B = (torch.randn(spec.n_adapters, out_f, spec.rank, device=dev) / 8).to(torch.bfloat16)
        pool = S.Pool(in_f, out_f, spec.rank, spec.n_adapters, S.SMLM_BF16, 0)
        for a in range(spec.n_adapters):
            pool.register(A[a], B[a], 2.0)
        sets.append((W, A, B, pool, torch.empty_like(pool.workspace(b, False))))
    for i in range(16):
        W, _, _, pool, ws = sets[i % 8]
        S.smlm_forward(pool.h, b, X, W, Y, None, ws)
    torch.cuda.synchronize()
    S.smlm_profile_enable(True)
    for kind in range(4):
        S.smlm_profile_read(kind)
    n = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        W, _, _, pool, ws = sets[i % 8]
        S.smlm_forward(pool.h, b, X, W, Y, None, ws)
    e1.record()
    torch.cuda.synchronize()
    gemm = S.smlm_profile_read(0)
    shr = S.smlm_profile_read(2)
    S.smlm_profile_enable(False)
    print(json.dumps({"proj": proj, "call_us": e0.elapsed_time(e1) / n * 1e3, "gemm_us": gemm[0] / gemm[1] * 1e3,
                      "shrink_us": shr[0] / max(shr[1], 1) * 1e3}), flush=True)
    for s_ in sets:
        s_[3].close()
