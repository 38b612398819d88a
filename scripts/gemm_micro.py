"""Micro-benchmark: the SMLM forward/backward tensor-core kernels vs cuBLAS (torch.matmul) on the
same shapes.  Prints one JSON line per case.  Not part of the product; a measurement aid."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dev = torch.device("cuda", 0)
    M = int(os.environ.get("M", "13448"))
    r = 16
    for (K, N) in [(4096, 14336), (14336, 4096), (4096, 4096), (4096, 1024)]:
        X = torch.randn(M, K, device=dev).to(torch.bfloat16)
        W = (torch.randn(N, K, device=dev) / math.sqrt(K)).to(torch.bfloat16)
        Y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        t_cublas = timeit(lambda: torch.matmul(X, W.t(), out=Y))
        pool = S.Pool(K, N, r, 8, S.SMLM_BF16, 0)
        A = (torch.randn(8, r, K, device=dev) / math.sqrt(K)).to(torch.bfloat16)
        B = (torch.randn(8, N, r, device=dev) / 8).to(torch.bfloat16)
        for i in range(8):
            pool.register(A[i], B[i], 2.0)
        lens = [M // 8] * 7 + [M - 7 * (M // 8)]
        res = {"K": K, "N": N, "M": M, "cublas_ms": t_cublas, "cublas_tflops": 2 * M * N * K / t_cublas / 1e9}
        for name, slots in (("base_only", [-1] * 8), ("lora", list(range(8)))):
            b = S.Batch(synth.batch_from_lengths(lens, slots, [2] * 8).offsets, slots, [2] * 8)
            ws = pool.workspace(b, False)
            t = timeit(lambda: S.smlm_forward(pool.h, b, X, W, Y, None, ws))
            res[f"smlm_{name}_ms"] = t
            res[f"smlm_{name}_tflops"] = 2 * M * N * K / t / 1e9
        # backward dX (all rows fine-tune)
        b = S.Batch(synth.batch_from_lengths(lens, list(range(8)), [0] * 8).offsets, list(range(8)), [0] * 8)
        dY = torch.randn(M, N, device=dev).to(torch.bfloat16)
        dX = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
        wsb = pool.workspace(b, True)
        t = timeit(lambda: S.smlm_backward(pool.h, b, X, W, dY, None, dX, 0, wsb))
        res["smlm_bwd_ms"] = t
        res["smlm_bwd_tflops_dx"] = 2 * M * N * K / t / 1e9
        t_cublas_bwd = timeit(lambda: torch.matmul(dY, W, out=dX))
        res["cublas_bwd_tflops"] = 2 * M * N * K / t_cublas_bwd / 1e9
        print(json.dumps(res), flush=True)
        pool.close()


if __name__ == "__main__":
    main()
