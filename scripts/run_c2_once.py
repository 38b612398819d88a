"""Tiny driver for profiling: a few C2 decode forward calls (q projection)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

k = int(os.environ.get("CFG", "2"))
proj = os.environ.get("PROJ", "q")
spec = synth.CONFIGS[k]
batch = synth.config_batch(k)
b = S.Batch.from_synth(batch)
in_f, out_f = synth.PROJ_SHAPES[proj]
dev = torch.device("cuda", 0)
X = torch.randn(batch.S, in_f, device=dev).to(torch.bfloat16)
W = (torch.randn(out_f, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
A = (torch.randn(spec.n_adapters, spec.rank, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
B = (torch.randn(spec.n_adapters, out_f, spec.rank, device=dev) / 8).to(torch.bfloat16)
pool = S.Pool(in_f, out_f, spec.rank, spec.n_adapters, S.SMLM_BF16, 0)
for a in range(spec.n_adapters):
    pool.register(A[a], B[a], 2.0)
Y = torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev)
ws = pool.workspace(b, False)
for _ in range(int(os.environ.get("N", "3"))):
    S.smlm_forward(pool.h, b, X, W, Y, None, ws)
torch.cuda.synchronize()
print("ok")
