"""C4 alm2map + map2alm from pageable numpy buffers (the C++ drop-in's std::vector path):
wall-clock ms per transform, median of 5 after a warm-up.  SHTC_COPY_THREADS sets the host
copy pool size."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_1106_0159_b200 import sht

g = sht.build_healpix_grid(2048)
ctx = sht.Context(0)
ctx.set_grid(g)
ctx.set_band(4096, 4096)
alm = sht.gaussian_alm(4096, 4096, 12345)
mp = np.empty(g.n_pix)
back = np.empty_like(alm)
ctx.alm2map(alm, out=mp)
ctx.map2alm(mp, out=back)
ta, tm = [], []
for _ in range(5):
    t0 = time.perf_counter()
    ctx.alm2map(alm, out=mp)
    t1 = time.perf_counter()
    ctx.map2alm(mp, out=back)
    t2 = time.perf_counter()
    ta.append((t1 - t0) * 1e3)
    tm.append((t2 - t1) * 1e3)
print(f"pageable alm2map {np.median(ta):.2f} ms map2alm {np.median(tm):.2f} ms sum {np.median(ta) + np.median(tm):.2f}")
