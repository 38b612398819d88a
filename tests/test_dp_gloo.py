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
