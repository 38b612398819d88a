"""Per-config measurements beside the main bench line (BASELINE.json configs[1], configs[2]):

  C2 decode : q,k,v,o forward over 256 one-row decode requests, 32 adapters r=16 (HBM-bound)
  C3 prefill: gate,up,down forward over 8 prefill segments of 512-2048 rows, 8 adapters r=64

Rotates 8 distinct weight sets so consecutive calls do not hit L2.  Reports per projection the
device time (CUDA events on the launching stream, median of iterations), the algorithmic bytes /
flops (SURVEY.md §8(d) rules) and the fraction of the measured HBM / bf16 peak.
"""
import json
import math
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
NSETS = 8


def run_config(k, iters=30, graphs=False, ranks=None):
    """ranks: optional per-adapter ranks (<= the config's) -- heterogeneous ranks in one pool
    (SURVEY f2): adapter a is registered with its first ranks[a] rank indices."""
    spec = synth.CONFIGS[k]
    dev = torch.device("cuda", 0)
    batch = synth.config_batch(k)
    b = S.Batch.from_synth(batch)
    r, U = spec.rank, spec.n_adapters
    slots = batch.slots
    uniq = sorted(set(int(s) for s in slots if s >= 0))
    out = []
    g = torch.Generator(device=dev)
    g.manual_seed(7 + k)
    total_ms = 0.0
    for p in spec.projections:
        in_f, out_f = synth.PROJ_SHAPES[p]
        X = torch.randn(batch.S, in_f, generator=g, device=dev).to(torch.bfloat16)
        Y = torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev)
        sets = []
        for _ in range(NSETS):
            W = (torch.randn(out_f, in_f, generator=g, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
            A = (torch.randn(U, r, in_f, generator=g, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
            B = (torch.randn(U, out_f, r, generator=g, device=dev) / (4 * math.sqrt(r))).to(torch.bfloat16)
            pool = S.Pool(in_f, out_f, r, U, S.SMLM_BF16, 0)
            keep = []
            for a in range(U):
                if ranks is None or ranks[a] == r:
                    pool.register(A[a], B[a], 2.0)
                else:
                    Aa, Ba = A[a][:ranks[a]].contiguous(), B[a][:, :ranks[a]].contiguous()
                    keep += [Aa, Ba]
                    pool.register(Aa, Ba, 2.0)
            ws = torch.empty(S.smlm_workspace_size(pool.h, b, False) + 256, dtype=torch.uint8, device=dev)
            sets.append((W, A, B, pool, ws, keep))
        st = torch.cuda.current_stream()

        def call(i):
            W, _, _, pool, ws, _ = sets[i % NSETS]
            S.smlm_forward(pool.h, b, X, W, Y, None, ws, st)
        for i in range(2 * NSETS):
            call(i)
        torch.cuda.synchronize()
        times = []
        for i in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            call(i)
            e1.record(st)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms_sync = statistics.median(times)
        # back-to-back: GPU time per call when the host stays ahead (events around the loop)
        import time as _t
        torch.cuda.synchronize()
        h0 = _t.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(iters):
            call(i)
        e1.record(st)
        host_us = (_t.perf_counter() - h0) / iters * 1e6
        e1.synchronize()
        ms = e0.elapsed_time(e1) / iters
        total_ms += ms
        Sx = batch.S
        nbytes = in_f * out_f * 2 + len(uniq) * r * (in_f + out_f) * 2 + Sx * (in_f + out_f) * 2
        lens = [int(batch.offsets[i + 1] - batch.offsets[i]) for i in range(batch.G)]
        rows_lora = sum(l for l, s in zip(lens, slots) if s >= 0)
        flops = 2.0 * Sx * in_f * out_f + 2.0 * rows_lora * r * (in_f + out_f)
        t_hbm = nbytes / (PEAKS["hbm_gbs"] * 1e9) * 1e3
        t_tc = flops / (PEAKS["bf16_tflops"] * 1e12) * 1e3
        out.append({"config": spec.name, "proj": p, "S": Sx, "ms": ms, "ms_isolated_call": ms_sync,
                    "host_us_per_call": host_us,
                    "alg_MiB": nbytes / 2**20, "alg_GFLOP": flops / 1e9,
                    "hbm_GBs": nbytes / ms / 1e6, "hbm_frac": nbytes / ms / 1e6 / PEAKS["hbm_gbs"],
                    "tflops": flops / ms / 1e9, "tensor_frac": flops / ms / 1e9 / PEAKS["bf16_tflops"],
                    "roofline_ms": max(t_hbm, t_tc), "roofline_frac": max(t_hbm, t_tc) / ms})
        for s_ in sets:
            s_[3].close()
    return out, total_ms


def c2_layer_step(iters=40, graphs=True):
    """C2 as a layer would issue it: q/k/v in ONE smlm_forward_multi call (they share X), then o
    (its input is the attention output) -- back to back over 8 rotated weight sets, and as a CUDA
    graph replay of 8 layer-steps.  Roofline units per SURVEY.md §8(d): the 4 projections' bytes."""
    k = 2
    spec = synth.CONFIGS[k]
    dev = torch.device("cuda", 0)
    batch = synth.config_batch(k)
    b = S.Batch.from_synth(batch)
    r, U = spec.rank, spec.n_adapters
    uniq = sorted(set(int(x) for x in batch.slots if x >= 0))
    g = torch.Generator(device=dev)
    g.manual_seed(17)
    in_f = 4096
    Xqkv = torch.randn(batch.S, in_f, generator=g, device=dev).to(torch.bfloat16)
    Xo = torch.randn(batch.S, in_f, generator=g, device=dev).to(torch.bfloat16)
    sets = []
    for _ in range(NSETS):
        layer = {}
        for p in ("q", "k", "v", "o"):
            _, out_f = synth.PROJ_SHAPES[p]
            W = (torch.randn(out_f, in_f, generator=g, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
            A = (torch.randn(U, r, in_f, generator=g, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
            B = (torch.randn(U, out_f, r, generator=g, device=dev) / (4 * math.sqrt(r))).to(torch.bfloat16)
            pool = S.Pool(in_f, out_f, r, U, S.SMLM_BF16, 0)
            if os.environ.get("DEC_KSPLIT"):   # measurement sweep of the decode split-K factor
                pool.set_option(S.SMLM_OPT_DEC_KSPLIT, int(os.environ["DEC_KSPLIT"]))
            for a in range(U):
                pool.register(A[a], B[a], 2.0)
            Y = torch.empty(batch.S, out_f, dtype=torch.bfloat16, device=dev)
            layer[p] = (W, A, B, pool, Y)
        sets.append(layer)
    qkv = [sets[0][p][3].h for p in ("q", "k", "v")]
    nws = max(S.smlm_workspace_size_multi(qkv, b), S.smlm_workspace_size(sets[0]["o"][3].h, b, False))
    ws = torch.empty(nws + 256, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def step(i):   # on the current stream (the capture stream inside the graph context)
        L = sets[i % NSETS]
        S.smlm_forward_multi([L[p][3].h for p in ("q", "k", "v")], b, Xqkv, [L[p][0] for p in ("q", "k", "v")],
                             [L[p][4] for p in ("q", "k", "v")], None, ws)
        S.smlm_forward(L["o"][3].h, b, Xo, L["o"][0], L["o"][4], None, ws)
    for i in range(2 * NSETS):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(iters):
        step(i)
    e1.record(st)
    e1.synchronize()
    ms_b2b = e0.elapsed_time(e1) / iters
    ms_graph = None
    if graphs:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=torch.cuda.Stream()):
            for i in range(NSETS):
                step(i)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        e0.record()
        reps = 10
        for _ in range(reps):
            gr.replay()
        e1.record()
        e1.synchronize()
        ms_graph = e0.elapsed_time(e1) / (reps * NSETS)
    roof_ms = 0.0
    for p in ("q", "k", "v", "o"):
        _, out_f = synth.PROJ_SHAPES[p]
        nbytes = in_f * out_f * 2 + len(uniq) * r * (in_f + out_f) * 2 + batch.S * (in_f + out_f) * 2
        flops = 2.0 * batch.S * in_f * out_f + 2.0 * batch.S * r * (in_f + out_f)
        roof_ms += max(nbytes / (PEAKS["hbm_gbs"] * 1e9), flops / (PEAKS["bf16_tflops"] * 1e12)) * 1e3
    for L in sets:
        for p in L:
            L[p][3].close()
    best = min(ms_b2b, ms_graph or 1e9)
    return {"config": "C2-decode layer-step (qkv fused + o)", "S": batch.S, "ms_back_to_back": ms_b2b,
            "ms_graph_replay": ms_graph, "roofline_ms": roof_ms, "rows_per_s": batch.S / (best / 1e3),
            "hbm_roofline_frac_b2b": roof_ms / ms_b2b,
            "hbm_roofline_frac_graph": None if ms_graph is None else roof_ms / ms_graph}


def adamw_step(layers=32, clip=1.0, iters=20, jobs=4):
    """AdamW over the C4 fine-tune adapters (4 adapters, r=16, 7 projections) of
    `layers` layers (kernels_opt.cu), one optimizer step PER fine-tune job (each job is its own
    trainer: own clip norm and step count, optim.py): `jobs` contiguous sub-ranges of one flat
    store, each a clip pass + a step launch.  34 algorithmic bytes/element (+4 with the clip
    pass); L2 flushed before every step."""
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    dev = torch.device("cuda", 0)
    n = 4 * synth.lora_param_count(16) * layers
    P, M, V, G = (torch.randn(n, device=dev) * 1e-3 for _ in range(4))
    V.abs_()
    PB = torch.empty(n, dtype=torch.bfloat16, device=dev)
    Wk = torch.empty(S.smlm_adamw_workspace_size() // 4, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for it in range(iters + 3):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for j in range(jobs):
            lo, hi = n * j // jobs // 8 * 8, (n * (j + 1) // jobs // 8 * 8 if j + 1 < jobs else n)
            S.smlm_adamw_step(P[lo:hi], M[lo:hi], V[lo:hi], G[lo:hi], PB[lo:hi], it + 1, 2e-5, max_grad_norm=clip,
                              zero_grad=True, ws=Wk)
        b.record()
        b.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    byts = n * (34 + (4 if clip > 0 else 0))
    del P, M, V, G, PB, flush
    return {"kernel": "smlm_adamw_step", "layers": layers, "n": n, "jobs": jobs, "clip": clip, "ms": ms, "alg_bytes": byts,
            "GB/s": byts / ms / 1e6, "hbm_peak_GB/s": hbm, "frac": byts / ms / 1e6 / hbm}


def main():
    if "--hetero" in sys.argv:
        # C3 (gate/up/down, 8 adapters at r=64) with uniform ranks vs mixed 64/32/16/8
        _, t_u = run_config(3, iters=10)
        _, t_h = run_config(3, iters=10, ranks=[64, 64, 32, 32, 16, 16, 8, 8])
        print(json.dumps({"config": "C3-prefill", "uniform_r64_ms": t_u, "hetero_64_32_16_8_ms": t_h,
                          "ratio": t_h / t_u}), flush=True)
        return
    if "--attention" in sys.argv:
        print(json.dumps(attention_step()), flush=True)
        return
    print(json.dumps(c2_layer_step(graphs="--c2-only" not in sys.argv)), flush=True)
    if "--c2-only" in sys.argv:
        return
    for k in (2, 3):
        rows, tot = run_config(k)
        for r in rows:
            print(json.dumps(r), flush=True)
        print(json.dumps({"config": synth.CONFIGS[k].name, "total_ms": tot,
                          "rows_per_s": synth.config_batch(k).S / (tot / 1e3),
                          "roofline_frac": sum(r["roofline_ms"] for r in rows) / tot}), flush=True)




def attention_step(iters=20, past=1024):
    """the Alg. 1 attention branch on the C4 batch structure at Llama-3-8B heads
    (32 query / 8 KV heads, d = 128): 4 fine-tune x 1024 + 8 prefill (512-2048, KV cache written) +
    128 decode rows each over a `past`-token cache.  Reports the prefill kernel's causal-attention
    tensor TF/s (4 * sum(L(L+1)/2) * d * Hq flops over the F/E/P segments) and the decode kernel's
    HBM GB/s (K + V cache bytes read), each timed alone with CUDA events (L2 flushed)."""
    from oracle.attention import DECODE, FINETUNE, PREFILL
    dev = torch.device("cuda", 0)
    batch = synth.config_batch(4)
    lens = np.diff(batch.offsets)
    modes = list(batch.modes)
    hq, hkv = 32, 8
    slots, pasts, slot = [], [], 0
    for L, m in zip(lens, modes):
        if m in (PREFILL, DECODE):
            slots.append(slot)
            slot += 1
        else:
            slots.append(-1)
        pasts.append(past if m == DECODE else 0)
    S_ = int(batch.S)
    g = torch.Generator(device=dev).manual_seed(5)
    Q = torch.randn(S_, hq, 128, generator=g, device=dev).to(torch.bfloat16)
    K = torch.randn(S_, hkv, 128, generator=g, device=dev).to(torch.bfloat16)
    V = torch.randn(S_, hkv, 128, generator=g, device=dev).to(torch.bfloat16)
    cap = max(2048, past + 8)
    Kc = torch.randn(slot, cap, hkv, 128, generator=g, device=dev).to(torch.bfloat16)
    Vc = torch.randn(slot, cap, hkv, 128, generator=g, device=dev).to(torch.bfloat16)
    O = torch.empty_like(Q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    offs = batch.offsets

    def timed(sel_modes):
        keep = [m in sel_modes for m in modes]
        lengths = [int(L) if k else 0 for L, k in zip(lens, keep)]
        b = S.AttnBatch(offs, modes, slots, pasts) if keep.count(True) == len(keep) else \
            S.AttnBatch(np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32), modes, slots, pasts)
        ws = torch.empty(max(S.smlm_attention_workspace_size(b, hq, hkv), 256), dtype=torch.uint8, device=dev)
        ts = []
        for it in range(iters + 3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            S.smlm_attention(b, Q, K, V, O, Kc, Vc, ws=ws)
            e1.record()
            e1.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    ms_pf = timed((FINETUNE, 1, PREFILL))
    ms_dec = timed((DECODE,))
    fe = [(int(L), m) for L, m in zip(lens, modes) if m != DECODE and L > 0]
    flops = sum(4.0 * L * (L + 1) / 2 * 128 * hq for L, _ in fe)
    # algorithmic decode bytes: each decode segment's cache (its past + its own rows) read once per
    # KV head -- the rows of one segment share the slot's K / V (not once per decode row)
    dec_bytes = sum((past + int(L)) * hkv * 128 * 2 * 2 for L, m in zip(lens, modes) if m == DECODE and L > 0)
    return {"workload": f"C4 batch, Llama-3-8B heads 32/8 d=128; decode rows over {past}-token caches",
            "prefill_ms": ms_pf, "prefill_tflops": flops / ms_pf / 1e9,
            "prefill_tensor_frac": flops / ms_pf / 1e9 / PEAKS["bf16_tflops"],
            "decode_ms": ms_dec, "decode_GBs": dec_bytes / ms_dec / 1e6,
            "decode_hbm_frac": dec_bytes / ms_dec / 1e6 / PEAKS["hbm_gbs"]}


if __name__ == "__main__":
    main()
