"""AdamW step (kernels_opt.cu) throughput against the HBM roofline: one JSON line per size.

Sizes: the C4 fine-tune adapters (4 adapters, r=16, all 7 Llama-3-8B projections) for one layer
and for all 32 layers.  Algorithmic bytes per element: read g, p, m, v (16) + write p, m, v (12)
+ bf16 p (2) + zeroed g (4) = 34 B; the clip pass reads g once more (+4 B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = float(peaks["hbm_gbs"])
dev = torch.device("cuda", 0)
per_layer = 4 * synth.lora_param_count(16)
for layers in (1, 32):
    n = per_layer * layers
    P, M, V, G = (torch.randn(n, device=dev) * 1e-3 for _ in range(4))
    V.abs_()
    PB = torch.empty(n, dtype=torch.bfloat16, device=dev)
    W = torch.empty(S.smlm_adamw_workspace_size() // 4, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for clip in (0.0, 1.0):
        ts = []
        for it in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            S.smlm_adamw_step(P, M, V, G, PB, it + 1, 2e-5, max_grad_norm=clip, zero_grad=True, ws=W)
            b.record()
            b.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        ts.sort()
        ms = ts[len(ts) // 2]
        byts = n * (34 + (4 if clip > 0 else 0))
        gbs = byts / ms / 1e6
        print(json.dumps({"kernel": "smlm_adamw_step", "layers": layers, "n": n, "clip": clip, "ms": round(ms, 4),
                          "alg_bytes": byts, "GB/s": round(gbs, 1), "hbm_peak_GB/s": hbm, "frac": round(gbs / hbm, 3)}))
