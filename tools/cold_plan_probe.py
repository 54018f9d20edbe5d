import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1106_0159_b200 import sht
g = sht.build_healpix_grid(2048)
a = sht.Context(0); a.set_grid(g); a.set_band(4096, 4096); a.plan()
alm = sht.gaussian_alm(4096, 4096, 1)
mp = a.alm2map(alm); b = a.map2alm(mp)
print("warm ctx done", flush=True)
for rep in range(2):
    t0 = time.perf_counter()
    c = sht.Context(0); c.set_grid(g); c.set_band(4096, 4096)
    t1 = time.perf_counter(); c.plan(); t2 = time.perf_counter()
    print(f"cold ctx {rep}: setup {1e3*(t1-t0):.1f} ms plan {1e3*(t2-t1):.1f} ms", flush=True)
    c.close()
