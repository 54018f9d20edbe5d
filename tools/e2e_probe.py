"""Breakdown of the host-buffer (e2e) transforms at C4: PCIe copy rates from pinned memory,
each transform's e2e time and stage timing, against the device-resident times."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import sht

nside, lmax = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 4096)))
dev = torch.device("cuda:0")
g = sht.build_healpix_grid(nside)
na = sht.alm_count(lmax, lmax)

# raw copy rates (skipped with E2E_SKIP_COPY=1)
import os
for nbytes in (() if os.environ.get("E2E_SKIP_COPY") else (na * 16, g.n_pix * 8)):
    h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True)),
                     ("both", None)):
        if fn is None:
            h2 = torch.empty_like(h).pin_memory()
            d2 = torch.empty_like(d)
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 5
            print(f"{name} {nbytes/1e6:.0f} MB each way: {dt*1e3:.2f} ms  {2*nbytes/dt/1e9:.1f} GB/s total", flush=True)
            continue
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"{name} {nbytes/1e6:.0f} MB: {dt*1e3:.2f} ms  {nbytes/dt/1e9:.1f} GB/s", flush=True)

ctx = sht.Context(0)
ctx.set_grid(g)
ctx.set_band(lmax, lmax)
ctx.plan()
if os.environ.get("E2E_PAGEABLE") == "1":  # plain numpy buffers, as the C++ drop-in's std::vectors
    alm = sht.gaussian_alm(lmax, lmax, 12345)
    mp = np.empty(g.n_pix)
    back = np.empty(na, np.complex128)
    mp.fill(0.0)
    back.fill(0.0)
else:
    alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 12345).view(np.float64)).pin_memory().numpy().view(np.complex128)
    mp = torch.empty(g.n_pix, dtype=torch.float64).pin_memory().numpy()
    back = torch.empty(2 * na, dtype=torch.float64).pin_memory().numpy().view(np.complex128)
for it in range(int(os.environ.get("E2E_ITERS", 4))):
    t0 = time.perf_counter()
    _, t1 = ctx.alm2map(alm, out=mp, timing=True)
    t_a = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, t2 = ctx.map2alm(mp, out=back, timing=True)
    t_m = time.perf_counter() - t0
    print(f"alm2map wall {t_a*1e3:.2f} ms {t1}", flush=True)
    print(f"map2alm wall {t_m*1e3:.2f} ms {t2}", flush=True)
ad = torch.from_numpy(alm.view(np.float64)).to(dev)
md = torch.empty(g.n_pix, dtype=torch.float64, device=dev)
bd = torch.empty_like(ad)
for it in range(3):
    print("dev alm2map", ctx.alm2map_dev(ad.data_ptr(), md.data_ptr(), timing=True))
    print("dev map2alm", ctx.map2alm_dev(md.data_ptr(), bd.data_ptr(), timing=True), flush=True)
