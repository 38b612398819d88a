import torch, time
dev = torch.device("cuda", 0)
N = 256 << 20
for ns in (1, 2, 3, 4):
    hs = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(ns)]
    ds = [torch.empty(N, dtype=torch.uint8, device=dev) for _ in range(ns)]
    sts = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(True); b = torch.cuda.Event(True)
        a.record()
        for i in range(ns):
            sts[i].wait_event(a)
            with torch.cuda.stream(sts[i]):
                ds[i].copy_(hs[i], non_blocking=True)
        for i in range(ns):
            torch.cuda.current_stream().wait_stream(sts[i])
        b.record(); b.synchronize()
        ms = a.elapsed_time(b)
    print("streams", ns, "GB/s", ns * N / ms / 1e6)
# D2H concurrently with H2D
h = torch.empty(N, dtype=torch.uint8).pin_memory(); d = torch.empty(N, dtype=torch.uint8, device=dev)
h2 = torch.empty(N, dtype=torch.uint8).pin_memory(); d2 = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t=time.time()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("h2d+d2h concurrent", 2*N/(time.time()-t)/1e9)
