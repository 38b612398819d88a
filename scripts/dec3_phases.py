"""Phase timeline of the single-launch decode kernel (SMLM_DEC3_DEBUG=1 writes per-CTA
globaltimer stamps to the workspace tail): t0 start, t1 base loads issued, t2 V published (W tiles),
t3 partials stored (bulk), t4 accumulator ready, t5 split arrivals complete, t6 Y stored."""
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
for proj in (os.environ.get("PROJ", "q,k").split(",")):
    in_f, out_f = synth.PROJ_SHAPES[proj]
    X = torch.randn(batch.S, in_f, device=dev).to(torch.bfloat16)
    W = (torch.randn(out_f, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
    A = (torch.randn(spec.n_adapters, spec.rank, in_f, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
    B = (torch.randn(spec.n_adapters, out_f, spec.rank, device=dev) / 8).to(torch.bfloat16)
    pool = S.Pool(in_f, out_f, spec.rank, spec.n_adapters, S.SMLM_BF16, 0)
    for a in range(spec.n_adapters):
        pool.register(A[a], B[a], 2.0)
    Y = torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev)
    ws = pool.workspace(b, False)
    n = S.smlm_workspace_size(pool.h, b, False)
    for _ in range(3):
        ws[n - 148 * 128:n].zero_()
        S.smlm_forward(pool.h, b, X, W, Y, None, ws)
        torch.cuda.synchronize()
    t = ws[n - 148 * 128:n].view(torch.int64).view(148, 16).cpu().numpy()
    used = t[:, 0] > 0
    t = t[used].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    wm = (t[:, 4] > 0) & (t[:, 15] == 0)
    out = {"proj": proj, "w_ctas": int(wm.sum()), "v_ctas": int((~wm).sum())}
    names = ["start", "loads_issued", "v_seen", "parts_stored", "acc_ready", "arrived", "stored", "xbar", "exp_issued", "mma_done"]
    for k, name in enumerate(names):
        col = rel[wm, k][t[wm, k] > 0]
        if len(col):
            out[name] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
    for k, name in [(1, "v_loads_issued"), (4, "v_acc_ready"), (3, "v_parts_stored"), (5, "v_arrived"), (6, "v_published")]:
        col = rel[~wm, k][t[~wm, k] > 0]
        if len(col):
            out[name] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
    print(json.dumps(out))
    pool.close()
