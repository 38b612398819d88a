"""Reference points for the decode shapes: cuBLAS (torch.matmul) on Y = X W^T with M=256 decode rows,
a 16 MiB device copy, and an empty-ish kernel -- measured back-to-back with CUDA events."""
import json
import math

import torch


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


dev = torch.device("cuda", 0)
X = torch.randn(256, 4096, device=dev).to(torch.bfloat16)
res = {}
for name, out in (("q", 4096), ("k", 1024)):
    Ws = [(torch.randn(out, 4096, device=dev) / 64).to(torch.bfloat16) for _ in range(8)]
    Y = torch.empty(256, out, device=dev, dtype=torch.bfloat16)
    i = [0]

    def mm():
        torch.matmul(X, Ws[i[0] % 8].t(), out=Y)
        i[0] += 1
    res[f"cublas_{name}_us"] = t(mm)
    res[f"cublas_{name}_GBs"] = (out * 4096 * 2 + 256 * (4096 + out) * 2) / res[f"cublas_{name}_us"] / 1e3
a = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
b = torch.empty_like(a)
res["copy16MiB_us"] = t(lambda: b.copy_(a))
z = torch.empty(1, device=dev)
res["tiny_kernel_us"] = t(lambda: z.add_(1))
print(json.dumps(res))
