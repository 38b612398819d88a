"""Phase timeline of the decode kernel in the bench's regime: C2 q/k/v (one smlm_forward_multi call)
and o over 8 rotated weight sets, back to back (no explicit flush: the rotation keeps W out of L2);
the stamps of the last q/k/v call and of the last o call.  Stamps (SMLM_DEC3_DEBUG, measure
library): 10 entry, 0 setup done, 12 shrink item published, 2 every item published (expand may
start), 1 K-loop loads issued,
8 expand issued, 9 last MMA, 4 accumulator ready, 3 partials stored, 5 splits arrived,
7 peers' partials loaded, 6 Y stored (medians over CTAs, us after the first CTA's entry)."""
import json
import os
import sys

os.environ["SMLM_DEC3_DEBUG"] = "1"
os.environ["SMLM_MEASURE_LIB"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

NS = 8
batch = synth.config_batch(2)
b = S.Batch.from_synth(batch)
dev = torch.device("cuda", 0)
spec = synth.CONFIGS[2]
X = torch.randn(batch.S, 4096, device=dev).to(torch.bfloat16)
Xo = torch.randn(batch.S, 4096, device=dev).to(torch.bfloat16)
sets = []
for _ in range(NS):
    pools, Ws, Ys, keep = [], [], [], []
    for p in ("q", "k", "v", "o"):
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
    sets.append((pools, Ws, Ys, keep))
hs0 = [p.h for p in sets[0][0][:3]]
n = max(S.smlm_workspace_size_multi(hs0, b), S.smlm_workspace_size(sets[0][0][3].h, b, False))
wsq = torch.zeros(n, dtype=torch.uint8, device=dev)
wso = torch.zeros(n, dtype=torch.uint8, device=dev)
nq = S.smlm_workspace_size_multi(hs0, b)
no = S.smlm_workspace_size(sets[0][0][3].h, b, False)
NSH = 640 * 4 * 4 * 8
names = {10: "entry", 0: "setup", 12: "shrink_item_done", 2: "all_published", 1: "kloop_issued", 8: "expand_issued", 9: "mma_done", 4: "acc_ready", 3: "parts_stored",
         5: "arrived", 7: "peers_loaded", 6: "y_stored"}


def step(i):
    pools, Ws, Ys, _ = sets[i % NS]
    S.smlm_forward_multi([p.h for p in pools[:3]], b, X, Ws[:3], Ys[:3], None, wsq)
    S.smlm_forward(pools[3].h, b, Xo, Ws[3], Ys[3], None, wso)


for i in range(3 * NS):
    step(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(3 * NS):
    step(i)
e1.record()
torch.cuda.synchronize()
res = {"layer_step_us_b2b": round(e0.elapsed_time(e1) * 1e3 / (3 * NS), 2)}
if "--graph" in sys.argv:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=torch.cuda.Stream()):
        for i in range(NS):
            step(i)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    res["layer_step_us_graph"] = round(e0.elapsed_time(e1) * 1e3 / (10 * NS), 2)
print(json.dumps(res))
absd = {}
for name, ws, nn in (("qkv", wsq, nq), ("o", wso, no)):
    t = ws[nn - 148 * 128:nn].view(torch.int64).view(148, 16).cpu().numpy()
    used = t[:, 10] > 0
    absd[name] = (int(t[used, 10].min()), int(t[used][:, 6].max()))

    t = t[used].astype(np.float64)
    rel = (t - t[:, 10].min()) / 1e3
    out = {"call": name, "ctas": int(used.sum())}
    for k, nm in names.items():
        col = rel[:, k][t[:, k] > 0]
        if len(col):
            out[nm] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
    print(json.dumps(out))
print(json.dumps({"qkv_span_us": (absd["qkv"][1] - absd["qkv"][0]) / 1e3, "gap_qkv_end_to_o_entry_us": (absd["o"][0] - absd["qkv"][1]) / 1e3,
                  "o_span_us": (absd["o"][1] - absd["o"][0]) / 1e3}))
