"""Small driver that launches every kernel of libsmlm.so once, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py

Covers: the CTA-pair forward GEMM (pre-shrink, short tiles, fine-tune V_save), the SIMT short-row
shrink, the U pass + dX GEMM + dA/dB token contraction (backward), the single-launch decode
kernel (one projection and q/k/v fused), the multi-projection pre-shrink of a mixed batch, the
1-CTA GEMM (SMLM_OPT_CTA_PAIR = 0), the fp32 test-mode kernels, the attention branch (prefill,
cache writes, split-KV decode) and the AdamW step.
No parity checks here (the tests do that): this only exercises the launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402
from synth import DECODE, EVAL, FINETUNE, PREFILL  # noqa: E402

dev = torch.device("cuda", 0)


def mixed(dtype, cta_pair=1):
    lengths = [200, 3, 1, 70, 1, 2, 130]
    modes = [FINETUNE, DECODE, DECODE, PREFILL, DECODE, EVAL, FINETUNE]
    slots = [0, 1, 2, 3, -1, 1, 2]
    tdt = torch.float32 if dtype == S.SMLM_FP32 else torch.bfloat16
    batch, w, X, dY = synth.random_case(4242, 256, 320, 16, 4, lengths, modes, slots, dtype=tdt)
    pool = S.Pool(256, 320, 16, 4, dtype, 0)
    pool.set_option(S.SMLM_OPT_CTA_PAIR, cta_pair)
    A = [a.to(dev) for a in w.A]
    B = [b.to(dev) for b in w.B]
    for i in range(4):
        pool.register(A[i], B[i], w.slot_scale[i])
    dA = torch.zeros(4, 16, 256, device=dev)
    dB = torch.zeros(4, 320, 16, device=dev)
    for i in range(4):
        pool.set_grad(i, dA[i], dB[i])
    b = S.Batch.from_synth(batch)
    Xd, Wd, dYd = X.to(dev), w.W.to(dev), dY.to(dev)
    V = torch.zeros(batch.S, 16, dtype=Xd.dtype, device=dev)
    dX = torch.zeros(batch.S, 256, dtype=Xd.dtype, device=dev)
    pool.forward(b, Xd, Wd, V_save=V)
    pool.backward(b, Xd, Wd, dYd, V, dX)
    pool.backward(b, Xd, Wd, dYd, None, dX, accumulate=True)   # V recompute
    torch.cuda.synchronize()
    pool.close()


def decode_and_multi():
    g = torch.Generator().manual_seed(3)
    rows = 96
    slots = torch.randint(-1, 6, (rows,), generator=g).tolist()
    batch, w, X, _ = synth.random_case(7, 512, 256, 16, 6, [1] * rows, [DECODE] * rows, slots)
    pools, Ws, Ys = [], [], []
    keep = []
    for p in range(3):
        pool = S.Pool(512, 256, 16, 6, S.SMLM_BF16, 0)
        A = [a.to(dev) for a in w.A]
        B = [bb.to(dev) for bb in w.B]
        keep += [A, B]
        for i in range(6):
            pool.register(A[i], B[i], w.slot_scale[i])
        pools.append(pool)
        Ws.append(w.W.to(dev))
        Ys.append(torch.empty(rows, 256, dtype=torch.bfloat16, device=dev))
    b = S.Batch.from_synth(batch)
    Xd = X.to(dev)
    pools[0].forward(b, Xd, Ws[0], Ys[0])
    ws = torch.empty(S.smlm_workspace_size_multi([p.h for p in pools], b) + 256, dtype=torch.uint8, device=dev)
    S.smlm_forward_multi([p.h for p in pools], b, Xd, Ws, Ys, None, ws)
    # mixed batch through the multi-projection pre-shrink
    lengths = [150, 90, 2, 1]
    mb, _, MX, _ = synth.random_case(9, 512, 256, 16, 6, lengths, [FINETUNE, PREFILL, DECODE, DECODE], [0, 2, 4, 5])
    mbb = S.Batch.from_synth(mb)
    Ym = [torch.empty(mb.S, 256, dtype=torch.bfloat16, device=dev) for _ in range(3)]
    ws = torch.empty(S.smlm_workspace_size_multi([p.h for p in pools], mbb) + 256, dtype=torch.uint8, device=dev)
    S.smlm_forward_multi([p.h for p in pools], mbb, MX.to(dev), Ws, Ym, None, ws)
    torch.cuda.synchronize()
    for p in pools:
        p.close()


def attention():
    # the Alg. 1 attention branch: a 300-row prefill (three query blocks, the last partial) with
    # KV-cache init, a 128-row fine-tune segment (one full block), and two decode rows
    g = torch.Generator().manual_seed(3)
    S_ = 430
    Q = torch.randn(S_, 8, 128, generator=g).to(torch.bfloat16).to(dev)
    K = torch.randn(S_, 2, 128, generator=g).to(torch.bfloat16).to(dev)
    V = torch.randn(S_, 2, 128, generator=g).to(torch.bfloat16).to(dev)
    Kc = torch.zeros(2, 512, 2, 128, dtype=torch.bfloat16, device=dev)
    Vc = torch.zeros_like(Kc)
    offs, modes, cs, past = [0, 300, 428, 429, 430], [PREFILL, FINETUNE, DECODE, DECODE], [0, -1, 0, 1], [0, 0, 300, 7]
    O = torch.empty(S_, 8, 128, dtype=torch.bfloat16, device=dev)
    S.smlm_attention(S.AttnBatch(offs, modes, cs, past), Q, K, V, O, Kc, Vc)
    torch.cuda.synchronize()


def adamw():
    n = 70001
    P, M, V, G = (torch.randn(n, device=dev) for _ in range(4))
    V.abs_()
    PB = torch.empty(n, dtype=torch.bfloat16, device=dev)
    W = torch.empty(S.smlm_adamw_workspace_size() // 4, device=dev)
    S.smlm_adamw_step(P, M, V, G, PB, 3, 1e-3, max_grad_norm=1.0, zero_grad=True, ws=W)
    torch.cuda.synchronize()


if __name__ == "__main__":
    mixed(S.SMLM_BF16)
    mixed(S.SMLM_BF16, cta_pair=0)
    mixed(S.SMLM_FP32)
    decode_and_multi()
    attention()
    adamw()
    print("sanitize_run: ok, launches", S.smlm_launch_count())
