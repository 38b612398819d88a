"""Tiny driver for ncu: the bench's C4 step restricted to ONE layer (layers=[0]), run twice (the
first is the warm-up).  Per step the CTA-pair GEMM launches are, in order: forward q/k/v (one
merged launch), o, gate/up (merged), down; backward down, gate/up (smlm_backward_multi), o,
q/k/v -- 8 per step, so `-k regex:smlm_gemm2 -s 8 -c 8` (forward: smlm_gemm2w_kernel, backward: smlm_gemm2_kernel) captures the second step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload(4, 0, dev)
st = torch.cuda.current_stream(dev)
for _ in range(int(os.environ.get("STEPS", "2"))):
    wl.step(st, layers=[0])
torch.cuda.synchronize()
print("ok")
