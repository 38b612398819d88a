"""Multi-process (gloo, world size 2) check of the data-parallel wiring on CPU.

Each rank owns its own seeded batch (different rows per rank), computes its fine-tune adapters'
dA/dB with the oracle into a paper_2511_00101_b200.dp.GradBucket, and all-reduces the bucket
with dp.AllReduce.  The reduced gradient must equal the oracle gradient over the union of both
ranks' fine-tune rows (SURVEY.md §8(e) parity)."""
import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from synth import DECODE, FINETUNE, PREFILL

IN, OUT, R, U = 48, 40, 4, 3
FT_SLOTS = [0, 2]


def _weights():
    return synth.draw_weights(torch.Generator().manual_seed(5), IN, OUT, R, U, dtype=torch.float64)


def _rank_batch(rank):
    g = torch.Generator().manual_seed(100 + rank)
    lengths = [3 + rank, 5, 2, 4 + 2 * rank]
    b = synth.batch_from_lengths(lengths, [0, 1, 2, 0], [FINETUNE, PREFILL, FINETUNE, DECODE])
    X = torch.randn(b.S, IN, generator=g, dtype=torch.float64)
    dY = torch.randn(b.S, OUT, generator=g, dtype=torch.float64)
    return b, X, dY


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2511_00101_b200.dp import AllReduce, GradBucket
    w = _weights()
    b, X, dY = _rank_batch(rank)
    _, dA, dB = oracle.backward(b, w.W, w.A, w.B, w.slot_scale, X, dY)
    bucket = GradBucket(FT_SLOTS, R, IN, OUT)
    for i, s in enumerate(FT_SLOTS):
        bucket.dA(i).copy_(torch.from_numpy(dA[s]))
        bucket.dB(i).copy_(torch.from_numpy(dB[s]))
    AllReduce(dist, "cpu")(bucket)
    torch.save(bucket.flat, os.path.join(out_dir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dp_allreduce_equals_union_oracle():
    import oracle
    from paper_2511_00101_b200.dp import GradBucket
    oracle.build()
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        flats = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    assert torch.equal(flats[0], flats[1])  # every rank holds the same reduced gradient
    # oracle over the union of both ranks' rows (segments concatenated)
    w = _weights()
    parts = [_rank_batch(r) for r in range(world)]
    lengths, slots, modes = [], [], []
    for b, _, _ in parts:
        lengths += np.diff(b.offsets).tolist()
        slots += b.slots.tolist()
        modes += b.modes.tolist()
    ub = synth.batch_from_lengths(lengths, slots, modes)
    X = torch.cat([p[1] for p in parts])
    dY = torch.cat([p[2] for p in parts])
    _, dA, dB = oracle.backward(ub, w.W, w.A, w.B, w.slot_scale, X, dY)
    ref = GradBucket(FT_SLOTS, R, IN, OUT)
    for i, s in enumerate(FT_SLOTS):
        ref.dA(i).copy_(torch.from_numpy(dA[s]))
        ref.dB(i).copy_(torch.from_numpy(dB[s]))
    assert torch.allclose(flats[0].double(), ref.flat.double(), rtol=1e-6, atol=1e-6)
    assert flats[0].abs().sum() > 0


def _worker_opt(rank, world, port, out_dir):
    """Masked DP training step: each rank's fine-tune gradient goes into the flat AdapterParams
    gradient (the layout the GPU optimizer uses), one all-reduce, then the AdamW update of the
    mean gradient -- applied here with the oracle (the CUDA step is covered by test_gpu_adamw)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from oracle import adamw as OA
    from paper_2511_00101_b200.dp import AllReduce
    from paper_2511_00101_b200.optim import AdapterParams
    w = _weights()
    b, X, dY = _rank_batch(rank)
    _, dA, dB = oracle.backward(b, w.W, w.A, w.B, w.slot_scale, X, dY)
    store = AdapterParams([(R, IN, OUT)] * len(FT_SLOTS), device="cpu")
    for i, s in enumerate(FT_SLOTS):
        store.load(i, w.A[s].float(), w.B[s].float())
        store.dA(i).copy_(torch.from_numpy(dA[s]))
        store.dB(i).copy_(torch.from_numpy(dB[s]))
    AllReduce(dist, "cpu")(store)
    p, _, _ = OA.adamw_step(store.master.numpy(), np.zeros(store.n), np.zeros(store.n), store.grad.numpy(), 1, 1e-3,
                            grad_scale=1.0 / world, max_norm=1.0)
    torch.save({"grad": store.grad, "p": torch.from_numpy(p)}, os.path.join(out_dir, f"opt{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_dp_flat_adapter_params_step():
    import oracle
    from paper_2511_00101_b200.optim import AdapterParams
    oracle.build()
    world = 2
    # layout: 8-element (16-byte) aligned pieces, disjoint views covering the buffer's data
    store = AdapterParams([(R, IN, OUT), (8, 64, 24)], device="cpu")
    assert all(a % 8 == 0 and b % 8 == 0 for a, b in store.offsets)
    assert store.dA(0).shape == (R, IN) and store.dB(1).shape == (24, 8) and store.A(1).dtype == torch.bfloat16
    store.grad.fill_(0)
    for k in range(2):
        store.dA(k).fill_(1.0)
        store.dB(k).fill_(1.0)
    assert int(store.grad.sum()) == R * IN + OUT * R + 8 * 64 + 24 * 8
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_opt, args=(world, _free_port(), d), nprocs=world, join=True)
        res = [torch.load(os.path.join(d, f"opt{r}.pt")) for r in range(world)]
    assert torch.equal(res[0]["grad"], res[1]["grad"]) and torch.equal(res[0]["p"], res[1]["p"])
    # the reduced flat gradient is the union-of-rows oracle gradient in the AdapterParams layout
    w = _weights()
    parts = [_rank_batch(r) for r in range(world)]
    lengths, slots, modes = [], [], []
    for b, _, _ in parts:
        lengths += np.diff(b.offsets).tolist()
        slots += b.slots.tolist()
        modes += b.modes.tolist()
    ub = synth.batch_from_lengths(lengths, slots, modes)
    _, dA, dB = oracle.backward(ub, w.W, w.A, w.B, w.slot_scale, torch.cat([p[1] for p in parts]),
                                torch.cat([p[2] for p in parts]))
    ref = AdapterParams([(R, IN, OUT)] * len(FT_SLOTS), device="cpu")
    for i, s in enumerate(FT_SLOTS):
        ref.dA(i).copy_(torch.from_numpy(dA[s]))
        ref.dB(i).copy_(torch.from_numpy(dB[s]))
    assert torch.allclose(res[0]["grad"].double(), ref.grad.double(), rtol=1e-6, atol=1e-6)
