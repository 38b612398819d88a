#!/usr/bin/env python
"""SMLM benchmark (BASELINE.json metric: "SMLM tokens/s at Llama-3-8B r=16 mixed batch; % of
HBM/tensor roofline").

One step = the SMLM work of L = 8 Llama-3-8B layers over the unified batch (BASELINE.json
configs[3], "C4": 4 fine-tune segments x 1024 rows + 8 prefill requests + 128 decode rows over a
64-adapter pool, r = 16): the forward of all 7 projections (q,k,v,o,gate,up,down) of layers
0..7, then the fine-tune backward (dX, dA, dB) of the 7 projections of layers 7..0 (SURVEY.md
§8(d) C5 step; every layer has its own weight set of 416 MiB, so no layer's weights are in L2
when it runs).  tokens/s = rows x L / step time = the per-layer throughput of SURVEY.md §8(d).
With --gpus N > 1 (torchrun, one process per GPU, NCCL): configs[4] "C5" -- every rank runs its
own C4-shaped batch over a replicated 256-adapter pool; the fine-tune dA/dB of each layer (one
flat fp32 bucket of the 7 projections, 20 MiB) are SUM all-reduced over NCCL on a side stream as
soon as that layer's backward is done, overlapping the next layer's backward; value = all ranks'
rows x L / max-over-ranks step time (weak scaling).

`--impl reference` times the fp64 CPU oracle (oracle/, test infrastructure) on a bounded row
sample of the same workload on this box's host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_00101_b200.dp import AllReduce, GradBucket  # noqa: E402

METRIC = "SMLM tokens/s at Llama-3-8B r=16 mixed batch; % of HBM/tensor roofline"
UNIT = "tokens/s"
N_LAYERS = 8              # layers (distinct weight sets, 416 MiB each > 126 MB L2) per step
FT_SLOTS = [0, 1, 2, 3]   # fine-tune adapters (C4/C5)
GROUP_OF = {"q": "attn", "k": "attn", "v": "attn", "o": "o", "gate": "mlp", "up": "mlp", "down": "down"}
# projections sharing X go through one smlm_forward_multi call (Alg. 1 P:331 joint QKV;
# SURVEY §8 f1): q/k/v, o, gate/up, down
FWD_GROUPS = [("q", "k", "v"), ("o",), ("gate", "up"), ("down",)]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained"),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        busy = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# workload
# ------------------------------------------------------------------------------------------
class Workload:
    def __init__(self, k: int, rank: int, dev: torch.device):
        from paper_2511_00101_b200 import smlm as S
        self.S = S
        self.k = k
        self.spec = synth.CONFIGS[k]
        self.dev = dev
        self.batch = synth.config_batch(k, rank)
        self.b = S.Batch.from_synth(self.batch)
        self.rows = self.batch.S
        self.ft_rows = len(self.batch.ft_rows())
        r = self.spec.rank
        U = self.spec.n_adapters
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + k)
        # activations: one input per projection group (q/k/v share X, gate/up share X)
        self.X = {}
        for grp, in_f in (("attn", 4096), ("o", 4096), ("mlp", 4096), ("down", 14336)):
            self.X[grp] = torch.randn(self.rows, in_f, generator=g, device=dev).to(torch.bfloat16)
        # V_save of the fine-tune rows is per layer (layer L's backward consumes layer L's forward V)
        self.dY, self.Y, self.dX = {}, {}, {}
        self.V = [{} for _ in range(N_LAYERS)]
        for p in synth.PROJECTIONS:
            in_f, out_f = synth.PROJ_SHAPES[p]
            self.dY[p] = torch.randn(self.rows, out_f, generator=g, device=dev).to(torch.bfloat16)
            self.Y[p] = torch.empty(self.rows, out_f, dtype=torch.bfloat16, device=dev)
            self.dX[p] = torch.empty(self.rows, in_f, dtype=torch.bfloat16, device=dev)
            for L in range(N_LAYERS):
                self.V[L][p] = torch.zeros(self.rows, r, dtype=torch.bfloat16, device=dev)
        # layer sets: base weights + adapter pools (replicated across ranks: same seeds)
        self.layers = []
        self.buckets = []   # one flat fp32 all-reduce bucket per layer (the 7 projections' FT dA/dB)
        for L in range(N_LAYERS):
            gw = torch.Generator(device=dev)
            gw.manual_seed(1000 + 10 * k + 100 * L)
            layer = {}
            for p in synth.PROJECTIONS:
                in_f, out_f = synth.PROJ_SHAPES[p]
                W = (torch.randn(out_f, in_f, generator=gw, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
                A = (torch.randn(U, r, in_f, generator=gw, device=dev) / math.sqrt(in_f)).to(torch.bfloat16)
                B = (torch.randn(U, out_f, r, generator=gw, device=dev) / (4 * math.sqrt(r))).to(torch.bfloat16)
                pool = S.Pool(in_f, out_f, r, U, S.SMLM_BF16, dev.index)
                for a in range(U):
                    assert pool.register(A[a], B[a], 2.0) == a
                # fine-tune adapters' grads: views of the layer's flat bucket (set below)
                bucket = None
                wsf = pool.workspace(self.b, False)
                wsf = torch.empty_like(wsf)
                wsb = torch.empty(S.smlm_workspace_size(pool.h, self.b, True) + 256, dtype=torch.uint8, device=dev)
                layer[p] = dict(W=W, A=A, B=B, pool=pool, grad=bucket, wsf=wsf, wsb=wsb)
            for grp in FWD_GROUPS:
                if len(grp) > 1:
                    hs = [layer[p]["pool"].h for p in grp]
                    n = S.smlm_workspace_size_multi(hs, self.b)
                    nb = S.smlm_workspace_size_backward_multi(hs, self.b)
                    layer[grp] = dict(h=hs, ws=torch.empty(n + 256, dtype=torch.uint8, device=dev),
                                      wsb=torch.empty(nb + 256, dtype=torch.uint8, device=dev))
            lb = LayerBucket(FT_SLOTS, r, dev)
            for p in synth.PROJECTIONS:
                layer[p]["grad"] = lb.bind(p, layer[p]["pool"])
            self.buckets.append(lb)
            self.layers.append(layer)

    def flops(self):
        """Algorithmic flops of one layer-step: forward 2 in out + 2 r (in+out)
        per row; fine-tune backward 2 in out + 4 r (in+out) per fine-tune row (no dW)."""
        r = self.spec.rank
        f = b = 0.0
        for p in synth.PROJECTIONS:
            in_f, out_f = synth.PROJ_SHAPES[p]
            f += self.rows * (2.0 * in_f * out_f + 2.0 * r * (in_f + out_f))
            b += self.ft_rows * (2.0 * in_f * out_f + 4.0 * r * (in_f + out_f))
        return f, b

    def fwd_gemm_flops(self, p):
        """Algorithmic flops of one forward tensor-core GEMM launch for projection p: the base
        product for every row plus the expand of every row that has an adapter (the shrink runs
        in the pre-shrink pass for long tiles and in the SIMT kernel for short rows)."""
        r = self.spec.rank
        in_f, out_f = synth.PROJ_SHAPES[p]
        lens = np.diff(self.batch.offsets)
        lora = self.batch.slots >= 0
        rows_lora = int(lens[lora].sum())
        return 2.0 * self.rows * in_f * out_f + 2.0 * rows_lora * r * out_f

    def step(self, stream, comm=None, layers=None):
        """One step: forward of every layer in order, then the fine-tune backward of every layer
        in reverse; comm(bucket) after each layer's backward (its all-reduce overlaps the next
        layer's backward).  The backward of a layer is 4 independent calls (down; gate+up and
        q+k+v through smlm_backward_multi: one dX GEMM launch per group; o): they alternate over
        two streams so one group's GEMM tail and small kernels overlap the next one's; both
        streams join before the layer's bucket is reduced."""
        S = self.S
        nvtx = torch.cuda.nvtx
        order = list(range(N_LAYERS)) if layers is None else list(layers)
        for L in order:
            nvtx.range_push(f"smlm fwd L{L}")   # NVTX ranges: phase markers for nsys / ncu --nvtx
            forward_groups(S, self.layers[L], self.b, lambda p: self.X[GROUP_OF[p]], self.Y, self.V[L], stream)
            nvtx.range_pop()
        if getattr(self, "_s2", None) is None:
            self._s2 = torch.cuda.Stream(self.dev)
        for L in reversed(order):
            nvtx.range_push(f"smlm bwd L{L}")
            layer = self.layers[L]
            ev = torch.cuda.Event()
            ev.record(stream)
            self._s2.wait_event(ev)
            for i, grp in enumerate(reversed(FWD_GROUPS)):
                backward_group(S, layer, self.b, self.X[GROUP_OF[grp[0]]], self.dY, self.V[L], self.dX, grp,
                               self._s2 if i % 2 == 1 else stream)
            ev2 = torch.cuda.Event()
            ev2.record(self._s2)
            stream.wait_event(ev2)
            nvtx.range_pop()
            if comm is not None:
                nvtx.range_push(f"smlm grad reduce L{L}")
                comm(self.buckets[L])
                nvtx.range_pop()


    def use_peer_reduce(self, dist):
        """Fused cross-rank reduction: every layer bucket becomes a view of this rank's
        slot in a dp.PeerReduce staging buffer; every pool fans its dA/dB out to the peers."""
        from paper_2511_00101_b200.dp import PeerReduce
        sizes = [lb.flat.numel() for lb in self.buckets]
        self._peer_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.peer = PeerReduce(dist, int(self._peer_off[-1]), self.dev)
        self.peer.set_fanout([self.layers[L][p]["pool"] for L in range(N_LAYERS) for p in synth.PROJECTIONS])
        self.bind_peer_slots(0)
        return self.peer

    def bind_peer_slots(self, parity):
        slot = self.peer.slot(parity)
        for L, lb in enumerate(self.buckets):
            lb.rebind(slot[int(self._peer_off[L]):int(self._peer_off[L + 1])], self.layers[L])


class LayerBucket:
    """One flat fp32 buffer per layer holding the fine-tune adapters' dA/dB of all 7 projections
    (one all-reduce bucket per layer, 20 MiB at C4/C5); each projection's grads are
    a dp.GradBucket-shaped view into it."""

    def __init__(self, slots, r, dev):
        self.slots = list(slots)
        n = sum(len(self.slots) * r * (i + o) for i, o in (synth.PROJ_SHAPES[p] for p in synth.PROJECTIONS))
        self.flat = torch.zeros(n, dtype=torch.float32, device=dev)
        self.r, self.off, self.views = r, 0, {}

    def rebind(self, flat, layer):
        """Move the bucket onto another buffer (e.g. a peer-reduction staging slot) and re-bind."""
        self.flat, self.off = flat, 0
        for p in synth.PROJECTIONS:
            self.bind(p, layer[p]["pool"])
            layer[p]["grad"] = self.views[p]

    def bind(self, p, pool):
        in_f, out_f = synth.PROJ_SHAPES[p]
        n = len(self.slots) * self.r * (in_f + out_f)
        gb = GradBucket(self.slots, self.r, in_f, out_f, flat=self.flat[self.off:self.off + n])
        self.off += n
        gb.bind(pool)
        self.views[p] = gb
        return gb


def backward_group(S, layer, b, X, dY, V, dX, grp, stream):
    """Backward of one projection group: smlm_backward_multi for projections that share X (one dX
    GEMM launch over all their n-tiles), smlm_backward for the others."""
    if len(grp) > 1:
        S.smlm_backward_multi(layer[grp]["h"], b, X, [layer[p]["W"] for p in grp], [dY[p] for p in grp],
                              [V[p] for p in grp], [dX[p] for p in grp], False, layer[grp]["wsb"], stream)
    else:
        e = layer[grp[0]]
        S.smlm_backward(e["pool"].h, b, X, e["W"], dY[grp[0]], V[grp[0]], dX[grp[0]], 0, e["wsb"], stream)


def forward_groups(S, layer, b, X_of, Y, V, stream, groups=None):
    """Forward of the projection groups: one smlm_forward_multi call per group of projections
    that share X (q/k/v, gate/up), smlm_forward for the others."""
    for grp in (groups or FWD_GROUPS):
        if len(grp) > 1:
            m = layer[grp]
            S.smlm_forward_multi(m["h"], b, X_of(grp[0]), [layer[p]["W"] for p in grp], [Y[p] for p in grp],
                                 [V[p] for p in grp], m["ws"], stream)
        else:
            e = layer[grp[0]]
            S.smlm_forward(e["pool"].h, b, X_of(grp[0]), e["W"], Y[grp[0]], V[grp[0]], e["wsf"], stream)


def _device_timed(fn, steps, stream):
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(steps):
        fn(i)
    end.record(stream)
    end.synchronize()
    return start.elapsed_time(end)


# ------------------------------------------------------------------------------------------
# oracle (reference arm / cpu_baseline) on a bounded row sample
# ------------------------------------------------------------------------------------------
def oracle_sample(k: int, n_sample: int, rank: int = 0):
    """Sub-batch of `n_sample` rows spread evenly over the workload's rows, keeping each row's
    segment (slot, mode); the oracle then runs forward over all 7 projections and the fine-tune
    backward (dX, dA, dB) over the sub-batch."""
    bt = synth.config_batch(k, rank)
    rs, rm = bt.row_slot(), bt.row_mode()
    idx = np.unique(np.linspace(0, bt.S - 1, n_sample).round().astype(np.int64))
    # segments of the sub-batch: consecutive sampled rows that came from the same segment
    seg_of = np.repeat(np.arange(bt.G), np.diff(bt.offsets))
    lengths, slots, modes = [], [], []
    for t in idx:
        g = seg_of[t]
        if lengths and seg_prev == g:
            lengths[-1] += 1
        else:
            lengths.append(1)
            slots.append(int(rs[t]))
            modes.append(int(rm[t]))
        seg_prev = g
    return synth.batch_from_lengths(lengths, slots, modes), idx


def run_oracle_step(sub, k, weights_cache):
    import oracle
    g = torch.Generator().manual_seed(77)
    n = sub.S
    for p in synth.PROJECTIONS:
        w = weights_cache[p]
        in_f, out_f = synth.PROJ_SHAPES[p]
        X = torch.randn(n, in_f, generator=g).to(torch.bfloat16)
        dY = torch.randn(n, out_f, generator=g).to(torch.bfloat16)
        oracle.forward(sub, w.W, w.A, w.B, w.slot_scale, X)
        if len(sub.ft_rows()):
            oracle.backward(sub, w.W, w.A, w.B, w.slot_scale, X, dY)


def oracle_weights(k):
    """Oracle-side weights: only the adapters the sample uses need values; shapes are full."""
    spec = synth.CONFIGS[k]
    cache = {}
    for p in synth.PROJECTIONS:
        in_f, out_f = synth.PROJ_SHAPES[p]
        g = torch.Generator().manual_seed(1000 + 10 * k + synth.PROJECTIONS.index(p))
        cache[p] = synth.draw_weights(g, in_f, out_f, spec.rank, spec.n_adapters)
    return cache


def time_oracle(k, n_sample, steps=1, threads=0):
    """Oracle rows/s on a row sample; threads: OpenMP threads (0 = all host cores)."""
    import oracle
    oracle.set_num_threads(threads)
    sub, _ = oracle_sample(k, n_sample)
    wc = oracle_weights(k)
    run_oracle_step(synth.batch_from_lengths([1], [0], [0]), k, wc)  # build + warm
    t0 = time.perf_counter()
    for _ in range(steps):
        run_oracle_step(sub, k, wc)
    dt = time.perf_counter() - t0
    used = oracle.num_threads()
    oracle.set_num_threads(0)
    return sub.S * steps / dt, dt, sub, used


# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-side", action="store_true", help="skip the C2 / C3 side measurements")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (production); gloo only to exercise the N>1 "
                    "path on a single-GPU box")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dp-reduce", default="fanout", choices=["fanout", "nccl"],
                    help="N > 1: fused peer-memory fan-out of dA/dB from the contraction kernel (SURVEY f3) or "
                         "an NCCL all-reduce per layer bucket")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="skip the per-kernel CUDA events (A/B check of their overhead)")
    ap.add_argument("--oracle-rows", type=int, default=48, help="cpu_baseline sample rows, all host cores")
    ap.add_argument("--oracle-rows-1t", type=int, default=6, help="cpu_baseline sample rows, 1 thread")
    ap.add_argument("--ref-rows", type=int, default=8, help="--impl reference sample rows per step")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(args.gpus, world)
    k = 4 if n == 1 else 5
    spec = synth.CONFIGS[k]

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        sub, _ = oracle_sample(k, args.ref_rows)
        wc = oracle_weights(k)
        for _ in range(args.warmup):
            run_oracle_step(sub, k, wc)
        samples = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run_oracle_step(sub, k, wc)
            samples.append(time.perf_counter() - t0)
        ms = 1000.0 * statistics.median(samples)
        val = sub.S / (ms / 1000.0)
        threads = oracle.num_threads()
        out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": n,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": spec.name, "sample_rows_per_step": sub.S},
               "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": f"{sub.S} rows evenly spread over the {spec.name} batch "
                                          f"(fp64 forward of 7 projections + fine-tune backward dX/dA/dB)"},
               "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    dist = None
    local = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2511_00101_b200 import smlm as S

    wl = Workload(k, rank, dev)
    stream = torch.cuda.current_stream(dev)
    comm = None
    peer = None
    dp_reduce = None
    if dist is not None:
        dp_reduce = args.dp_reduce
        if dp_reduce == "fanout":
            # the dA/dB contraction stores every gradient into its slot of every peer's
            # staging buffer over NVLink; the step ends when all ranks' slots have arrived
            try:
                peer = wl.use_peer_reduce(dist)
            except Exception as ex:   # e.g. no peer access between the devices: NCCL instead
                print(f"[bench] fan-out reduction unavailable ({ex!r:.120}); using NCCL all-reduce", file=sys.stderr)
                dp_reduce = "nccl"
        if dp_reduce == "nccl":
            allreduce = AllReduce(dist, dev)

            def comm(bucket):
                allreduce(bucket, stream)

    def one_step(i):
        if peer is not None:
            wl.bind_peer_slots(i % 2)
        wl.step(stream, comm)
        if comm is not None:
            allreduce.join(stream)
        if peer is not None:
            peer.signal(stream)
            peer.wait(stream)

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()

    # ---- the timed region: K steps, an event after each (all streams joined at a step's end);
    # no per-launch events in here (they would serialise programmatic dependent launch) ----
    launches0 = S.smlm_launch_count()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for i in range(args.steps):
        one_step(i)
        ev[i + 1].record(stream)
    ev[-1].synchronize()
    torch.cuda.synchronize()
    launches = S.smlm_launch_count() - launches0
    clk = clocks.stop()
    ms_total = ev[0].elapsed_time(ev[-1])
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    if dist is not None:
        t = torch.tensor([ms_total] + per_step, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, per_step = float(t[0].item()), [float(x) for x in t[1:].tolist()]
        dist.barrier()
    ms = ms_total / args.steps
    value = n * wl.rows * N_LAYERS / (ms / 1000.0)
    q = np.percentile(np.array(per_step), [10, 50, 90])
    step_stats = {"p10_ms": float(q[0]), "p50_ms": float(q[1]), "p90_ms": float(q[2]),
                  "mean_ms": ms, "note": "per-step CUDA events on the launching stream, max over ranks"}

    # ---- roofline of the dominant kernel (the forward tensor-core GEMM): a second pass of K
    # steps with CUDA events around each of its launches on the launching stream ----
    prof = {kind: (0.0, 0) for kind in range(4)}
    ms_prof = None
    if not args.no_kernel_timing:
        S.smlm_profile_enable(1)
        for kind in range(4):
            S.smlm_profile_read(kind)
        torch.cuda.synchronize()
        ms_prof = _device_timed(one_step, args.steps, stream)
        torch.cuda.synchronize()
        prof = {kind: S.smlm_profile_read(kind) for kind in range(4)}
        S.smlm_profile_enable(False)
    peaks = _peaks()
    fwd_ms, fwd_n = prof[0]
    fwd_flops = sum(wl.fwd_gemm_flops(p) for p in synth.PROJECTIONS) * N_LAYERS * args.steps
    achieved = fwd_flops / (fwd_ms / 1000.0) / 1e12 if fwd_ms > 0 else 0.0
    # denominator: the burst cuBLAS peak when the timed region ran at max SM clock, else (power
    # cap active, clocks below max) the sustained one measured under the same cap; both reported
    peak_b = peaks["bf16"]
    peak_s = peaks["bf16_sustained"] or peaks["bf16"]
    at_max = bool(clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"])
    peak = peak_b if at_max else peak_s
    traffic = None
    ncu_sum = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu_sum):
        try:
            with open(ncu_sum) as f:
                traffic = json.load(f).get("fwd_gemm_dram_bytes_per_launch")
        except Exception:
            traffic = None
    f_alg, b_alg = wl.flops()
    step_tflops = (f_alg + b_alg) * N_LAYERS / (ms / 1000.0) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "kernel": "smlm_gemm2w_kernel<fwd> (tcgen05 cta_group::2; 256 x 512 items over both TMEM halves, full W tiles + s*V expand K-block, TMA-store epilogue)",
                "peak_source": peaks["source"] + (" bf16_tflops (burst: the timed region ran at max SM clock)" if at_max
                                                  else " bf16_tflops_sustained (the timed region ran below max SM "
                                                       "clock under the power cap)"),
                "frac_burst": achieved / peak_b if peak_b else None, "peak_burst": peak_b,
                "frac_sustained": achieved / peak_s if peak_s else None, "peak_sustained": peak_s,
                "launches": fwd_n, "avg_launch_ms": fwd_ms / max(fwd_n, 1),
                "share_of_step": fwd_ms / ms_prof if ms_prof else None,
                "timing": "per-launch CUDA events in a second pass of the same K steps (the graded timed "
                          "region has none)",
                "step_alg_tflops": step_tflops, "step_frac": step_tflops / peak,
                "step_frac_burst": step_tflops / peak_b, "step_frac_sustained": step_tflops / peak_s}

    # ---- end to end: host buffers through the public API ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(wl, stream, max(4, min(args.steps, 8)), n, dist)

    # the headline workload's device memory (8 layer sets, ~20 GB) is released before the side
    # measurements, which then run on their own allocations as a standalone run would
    wl_rows, wl_ft_rows = wl.rows, wl.ft_rows
    del wl
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---- the other BASELINE.json configs as side measurements (rank 0, N=1): C2 decode layer-step
    # (q/k/v in one smlm_forward_multi launch + o; CUDA-graph replay) and C3 prefill ----
    side = None
    if rank == 0 and n == 1 and not args.no_side:
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            import bench_configs as bc
            at = bc.attention_step()   # first: the smallest side workloads on a clean heap
            c2 = bc.c2_layer_step()
            rows3, tot3 = bc.run_config(3, iters=10)
            side = {"C2_decode": {"workload": c2["config"], "rows": c2["S"], "ms_graph_replay": c2["ms_graph_replay"],
                                  "ms_back_to_back": c2["ms_back_to_back"], "rows_per_s": c2["rows_per_s"],
                                  "hbm_roofline_frac": c2["hbm_roofline_frac_graph"],
                                  "hbm_roofline_frac_back_to_back": c2["hbm_roofline_frac_b2b"],
                                  "roofline_ms": c2["roofline_ms"], "bound": "hbm"},
                    "C3_prefill": {"workload": synth.CONFIGS[3].name + ": gate, up, down", "ms": tot3,
                                   "rows_per_s": synth.config_batch(3).S / (tot3 / 1e3),
                                   "tensor_roofline_frac": sum(r["roofline_ms"] for r in rows3) / tot3,
                                   "bound": "tensor"}}
            side["F4_attention"] = {"workload": at["workload"], "prefill_ms": at["prefill_ms"],
                                    "prefill_tflops": at["prefill_tflops"],
                                    "prefill_tensor_roofline_frac": at["prefill_tensor_frac"],
                                    "decode_ms": at["decode_ms"], "decode_GBs": at["decode_GBs"],
                                    "decode_hbm_roofline_frac": at["decode_hbm_frac"]}
            ad = bc.adamw_step(layers=32)
            side["F3_adamw"] = {"workload": "AdamW step (clip 1.0 per job) over the C4 fine-tune adapters: 4 jobs x "
                                            "r=16 x 7 projections x 32 layers, one step per job", "n": ad["n"],
                                "ms": ad["ms"],
                                "GB/s": ad["GB/s"], "hbm_roofline_frac": ad["frac"], "bound": "hbm",
                                "alg_bytes_per_element": 38}
        except Exception as ex:   # side measurements never break the headline line
            side = {"error": repr(ex)[:200]}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        v, dt, sub, threads = time_oracle(k, args.oracle_rows, 1)
        v1, dt1, sub1, _ = time_oracle(k, args.oracle_rows_1t, 1, threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{sub.S} rows evenly spread over the {spec.name} batch; fp64 forward of 7 projections "
                         f"+ fine-tune backward (dX, dA, dB) = one layer-step of those rows; {dt:.1f} s",
               "single_thread": {"value": v1, "unit": UNIT, "cores": 1,
                                 "sample": f"{sub1.S} rows, same recipe; {dt1:.1f} s"}}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": {"workload": spec.name + ": Llama-3-8B projections q,k,v,o,gate,up,down; r=16; "
                          f"{spec.n_adapters} adapters; 4 fine-tune x 1024 rows (fwd+bwd) + 8 prefill "
                          "(512-2048) + 128 decode rows",
                          "rows_per_layer_per_gpu": wl_rows, "finetune_rows": wl_ft_rows, "rank": spec.rank,
                          "adapters": spec.n_adapters, "parallelism": f"dp{n}", "layers_per_step": N_LAYERS,
                          "l2": f"inputs larger than L2: every layer of the step has its own weight set "
                                f"(416 MiB each, {N_LAYERS} per step)",
                          "step": f"forward of the 7 projections of layers 0..{N_LAYERS - 1}, then the fine-tune "
                                  f"backward of layers {N_LAYERS - 1}..0"
                                  + ((" with one NCCL all-reduce of the layer's fine-tune dA/dB (20 MiB fp32 bucket) "
                                      "per layer, overlapping the next layer's backward") if dp_reduce == "nccl" else
                                     (" with the fine-tune dA/dB stored into every peer's staging slot by the dA/dB "
                                      "contraction kernel itself (NVLink peer memory), then a device-side wait for all "
                                      "ranks' slots") if dp_reduce == "fanout" else ""),
                          "dp_reduce": dp_reduce,
                          "tokens_per_s": "rows x layers / step time (per-layer throughput, SURVEY §8(d))"},
               "step_stats": step_stats,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
               "clocks": clk, "configs": side}
        print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(wl, stream, steps, n, dist):
    """Same step through the public API with HOST buffers: every step copies the step's inputs
    (X per projection group for every row; dY of the fine-tune rows) from pinned host memory and
    reads back the step's results: every layer's fine-tune dA/dB (what the optimizer consumes) and
    Y of the decode rows of every projection of the last layer (what the serving loop consumes).
    Intermediates that stay on the device in a real model (other layers' activations, prefill /
    fine-tune Y, dX) are not copied.

    Pipelined like a serving/training loop would be: device buffers are double-buffered, H2D of
    step i+1 runs on its own stream while step i computes, and each projection's outputs are read
    back on a D2H stream as soon as that projection finishes.  Timed from the first H2D to the
    last D2H with CUDA events (all copies and kernels inside the timed region)."""
    S = wl.S
    ft = wl.ft_rows  # fine-tune segments come first (row order F, E, P, D)
    dev = wl.dev
    hX = {g: torch.empty_like(x, device="cpu").pin_memory() for g, x in wl.X.items()}
    hdY = {p: torch.empty(ft, y.shape[1], dtype=y.dtype).pin_memory() for p, y in wl.dY.items()}
    # decode rows are the trailing DECODE segments (row order F, E, P, D)
    dec0 = int(wl.batch.offsets[int(np.argmax(wl.batch.modes == synth.DECODE))]) if np.any(
        wl.batch.modes == synth.DECODE) else wl.rows
    hY = {p: torch.empty(wl.rows - dec0, y.shape[1], dtype=y.dtype).pin_memory() for p, y in wl.Y.items()}
    hG = [torch.empty_like(b.flat, device="cpu").pin_memory() for b in wl.buckets]
    for g in hX:
        hX[g].copy_(wl.X[g].cpu())
    for p in hdY:
        hdY[p].copy_(wl.dY[p][:ft].cpu())
    h2d = sum(t.numel() * t.element_size() for t in hX.values()) + sum(t.numel() * t.element_size() for t in hdY.values())
    d2h = sum(t.numel() * t.element_size() for t in hY.values()) + sum(t.numel() * t.element_size() for t in hG)
    # double-buffered device tensors: [0] = the workload's own, [1] = a second set
    Xb = [wl.X, {g: torch.empty_like(x) for g, x in wl.X.items()}]
    dYb = [wl.dY, {p: torch.empty_like(y) for p, y in wl.dY.items()}]
    Yb = [wl.Y, {p: torch.empty_like(y) for p, y in wl.Y.items()}]
    dXb = [wl.dX, {p: torch.empty_like(x) for p, x in wl.dX.items()}]
    Vb = [wl.V, [{p: torch.zeros_like(v) for p, v in VL.items()} for VL in wl.V]]
    s_h2d = torch.cuda.Stream(dev)
    s_h2d2 = torch.cuda.Stream(dev)   # second copy engine for the input stream
    s_d2h = torch.cuda.Stream(dev)
    in_ready = [torch.cuda.Event(), torch.cuda.Event()]
    diag = [] if os.environ.get("BENCH_E2E_DIAG") else None   # per-step copy/compute timeline (stderr)
    in_free = [None, None]
    out_done = [None, None]

    def issue_inputs(i):
        b = i % 2
        if in_free[b] is not None:
            s_h2d.wait_event(in_free[b])
            s_h2d2.wait_event(in_free[b])
        with torch.cuda.stream(s_h2d):
            for g in hX:
                Xb[b][g].copy_(hX[g], non_blocking=True)
        with torch.cuda.stream(s_h2d2):
            for p in hdY:
                dYb[b][p][:ft].copy_(hdY[p], non_blocking=True)
        if diag is not None:
            e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e1.record(s_h2d)
            e2.record(s_h2d2)
            diag.append(("h2d_x_end", i, e1))
            diag.append(("h2d_dy_end", i, e2))
        s_h2d.wait_stream(s_h2d2)
        in_ready[b].record(s_h2d)

    if getattr(wl, "_s2", None) is None:
        wl._s2 = torch.cuda.Stream(dev)

    def compute(i):
        b = i % 2
        if getattr(wl, "peer", None) is not None:
            wl.bind_peer_slots(wl.peer.steps % 2)
        stream.wait_event(in_ready[b])
        if out_done[b] is not None:
            stream.wait_event(out_done[b])
        if diag is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            diag.append(("compute_start", i, e))
        for L in range(N_LAYERS):
            layer = wl.layers[L]
            for grp in FWD_GROUPS:
                forward_groups(S, layer, wl.b, lambda p: Xb[b][GROUP_OF[p]], Yb[b], Vb[b][L], stream, [grp])
                if L == N_LAYERS - 1:
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    s_d2h.wait_event(ev)
                    with torch.cuda.stream(s_d2h):
                        for p in grp:
                            hY[p].copy_(Yb[b][p][dec0:], non_blocking=True)
        for L in reversed(range(N_LAYERS)):
            layer = wl.layers[L]
            ev = torch.cuda.Event()
            ev.record(stream)
            wl._s2.wait_event(ev)
            for j, grp in enumerate(reversed(FWD_GROUPS)):
                backward_group(S, layer, wl.b, Xb[b][GROUP_OF[grp[0]]], dYb[b], Vb[b][L], dXb[b], grp,
                               wl._s2 if j % 2 else stream)
            ev = torch.cuda.Event()
            ev.record(wl._s2)
            stream.wait_event(ev)
            if dist is not None and getattr(wl, "peer", None) is None:
                dist.all_reduce(wl.buckets[L].flat, op=dist.ReduceOp.SUM)
            ev = torch.cuda.Event()
            ev.record(stream)
            s_d2h.wait_event(ev)
            with torch.cuda.stream(s_d2h):
                hG[L].copy_(wl.buckets[L].flat, non_blocking=True)
        if getattr(wl, "peer", None) is not None:
            wl.peer.signal(stream)
            wl.peer.wait(stream)
        ev = torch.cuda.Event(enable_timing=diag is not None)
        ev.record(stream)
        in_free[b] = ev
        if diag is not None:
            diag.append(("compute_end", i, ev))
        od = torch.cuda.Event()
        od.record(s_d2h)
        out_done[b] = od

    # warm-up one pipelined pass, then time `steps` steps end to end
    issue_inputs(0)
    compute(0)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s_h2d)
    issue_inputs(0)
    for i in range(steps):
        if i + 1 < steps:
            issue_inputs(i + 1)
        compute(i)
    s_d2h.wait_stream(stream)
    t1.record(s_d2h)
    t1.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if diag is not None:
        for name, i, e in diag:
            if e.query():
                try:
                    print(f"[e2e diag] step {i} {name} {t0.elapsed_time(e):.2f} ms", file=sys.stderr)
                except RuntimeError:
                    pass
    if dist is not None:
        t = torch.tensor([ms], device=wl.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del Xb, dYb, Yb, dXb, Vb
    return {"value": n * wl.rows * N_LAYERS / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms,
            "h2d": "X of every row (4 activation groups) + dY of the fine-tune rows, once per step",
            "d2h": f"fine-tune dA/dB of the 7 projections of all {N_LAYERS} layers + Y of the decode rows "
                   "(last layer)",
            "pipelining": "double-buffered; H2D of step i+1 and per-layer D2H overlap step i's kernels"}


if __name__ == "__main__":
    main()
