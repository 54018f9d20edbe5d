"""PCIe copy rate between pinned host memory and the GPU (403 MB, the C4 map) with the copy
split over 1, 2, 4 and 8 streams: one copy engine per direction already saturates the link."""
import torch, time
dev = torch.device("cuda:0")
n = 403 * 1000 * 1000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device=dev)
for k in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"D2H {k} streams: {n*8/dt/1e9:.1f} GB/s", flush=True)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D {k} streams: {n*8/dt/1e9:.1f} GB/s", flush=True)
