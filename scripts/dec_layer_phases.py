"""Phase timeline of the fused q/k/v decode launch (smlm_forward_multi) at C2 shapes."""
import json
import math
import os
import sys

os.environ["SMLM_DEC3_DEBUG"] = "1"
os.environ["SMLM_MEASURE_LIB"] = "1"   # build.py --measure
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

batch = synth.config_batch(2)
b = S.Batch.from_synth(batch)
dev = torch.device("cuda", 0)
spec = synth.CONFIGS[2]
X = torch.randn(batch.S, 4096, device=dev).to(torch.bfloat16)
pools, Ws, Ys, keep = [], [], [], []
for p in ("q", "k", "v"):
    _, out_f = synth.PROJ_SHAPES[p]
    W = (torch.randn(out_f, 4096, device=dev) / 64).to(torch.bfloat16)
    A = (torch.randn(spec.n_adapters, spec.rank, 4096, device=dev) / 64).to(torch.bfloat16)
    B = (torch.randn(spec.n_adapters, out_f, spec.rank, device=dev) / 8).to(torch.bfloat16)
    pool = S.Pool(4096, out_f, spec.rank, spec.n_adapters)
    for a in range(spec.n_adapters):
        pool.register(A[a], B[a], 2.0)
    pools.append(pool)
    Ws.append(W)
    Ys.append(torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev))
    keep += [A, B]
n = S.smlm_workspace_size_multi([p.h for p in pools], b)
ws = torch.empty(n, dtype=torch.uint8, device=dev)
for _ in range(3):
    ws[n - 148 * 128:n].zero_()
    S.smlm_forward_multi([p.h for p in pools], b, X, Ws, Ys, None, ws)
    torch.cuda.synchronize()
t = ws[n - 148 * 128:n].view(torch.int64).view(148, 16).cpu().numpy()
used = t[:, 0] > 0
t = t[used].astype(np.float64)
rel = (t - t[:, 0].min()) / 1e3
wm = (t[:, 4] > 0) & (t[:, 15] == 0)
names = ["start", "loads_issued", "v_seen", "parts_stored", "acc_ready", "arrived", "stored"]
out = {"w_ctas": int(wm.sum()), "v_ctas": int((~wm).sum())}
for k, name in enumerate(names):
    col = rel[wm, k][t[wm, k] > 0]
    if len(col):
        out[name] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
for k, name in [(1, "v_loads_issued"), (4, "v_acc_ready"), (3, "v_parts_stored"), (5, "v_arrived"), (6, "v_published")]:
    col = rel[~wm, k][t[~wm, k] > 0]
    if len(col):
        out[name] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
print(json.dumps(out))
