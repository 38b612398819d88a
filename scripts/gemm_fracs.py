"""Live (CUDA-event) average time of the forward and backward CTA-pair GEMM launches of the C4
step and their algorithmic tensor-core fraction (diagnostic; bench.py reports the forward one)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload(4, synth.CONFIGS[4].rank, dev)
st = torch.cuda.current_stream()
for i in range(4):
    wl.step(st)
torch.cuda.synchronize()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
for kind, name in ((0, "fwd"), (1, "bwd")):
    S.smlm_profile_enable(1 << kind)
    S.smlm_profile_read(kind)
    for i in range(6):
        wl.step(st)
    torch.cuda.synchronize()
    ms, n = S.smlm_profile_read(kind)
    S.smlm_profile_enable(0)
    f, b = wl.flops()
    fl = (sum(wl.fwd_gemm_flops(p) for p in synth.PROJECTIONS) if kind == 0 else b) * 6 * bench.N_LAYERS
    print(json.dumps({"gemm": name, "launches": n, "ms_total": ms, "tflops": fl / ms / 1e9,
                      "frac_sustained": fl / ms / 1e9 / peaks["bf16_tflops_sustained"]}))
