"""Phase timeline of the decode main kernel (SMLM_DEC3_DEBUG stamps, measure library) for q alone
and for the fused q/k/v call at C2 shapes; medians over the CTAs with work, us after the first
CTA's entry.  Stamps: 10 entry, 0 setup done, 11 shrink-prologue loads issued, 12 shrink prologue
done (slabs published), 1 K-loop loads issued, 2 every slab published (expand may start), 8 expand loads issued, 9 last MMA issued, 4 accumulator ready,
3 partials stored, 5 all splits arrived, 7 peers' partials loaded, 6 Y stored."""
import json
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
names = {10: "entry", 0: "setup", 11: "shrink_issued", 13: "sh_chunks_read", 14: "sh_peer_half", 15: "sh_fenced", 12: "shrink_published", 1: "kloop_issued", 2: "shrink_done", 8: "expand_issued", 9: "mma_done",
         4: "acc_ready", 3: "parts_stored", 5: "arrived", 7: "peers_loaded", 6: "y_stored"}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for npj in (1, 3):
    hs = [p.h for p in pools[:npj]]
    n = S.smlm_workspace_size_multi(hs, b)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(4):
        ws[n - 148 * 128:n].zero_()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.smlm_forward_multi(hs, b, X, Ws[:npj], Ys[:npj], None, ws)
        e1.record()
        torch.cuda.synchronize()
    t = ws[n - 148 * 128:n].view(torch.int64).view(148, 16).cpu().numpy()
    used = t[:, 10] > 0
    t = t[used].astype(np.float64)
    rel = (t - t[:, 10].min()) / 1e3
    out = {"proj": npj, "ctas": int(used.sum()), "event_us": round(e0.elapsed_time(e1) * 1e3, 2)}
    for k, name in names.items():
        col = rel[:, k][t[:, k] > 0]
        if len(col):
            out[name] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
    print(json.dumps(out))
