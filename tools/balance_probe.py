"""Executed-work balance of the m-distribution (reference assign_m min-max pairs) at C4: each
worker's plan on one GPU, executed stream-steps per worker, max / mean for W = 2, 4, 8."""
import sys
sys.path.insert(0, ".")
from paper_1106_0159_b200 import sht

nside, lmax = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 4096)))
g = sht.build_healpix_grid(nside)
for W in (2, 4, 8):
    layout = sht.WorkerLayout.create(g, lmax, W)
    ex = []
    for r in range(W):
        ctx = sht.Context(0)
        ctx.set_grid(g)
        ctx.set_band(lmax, lmax, layout.m_sets[r])
        ctx.plan()
        ex.append(ctx.plan_stats()["executed"])
        ctx.close()
    mean = sum(ex) / W
    print(f"W={W} executed per worker (G) {[round(e / 1e9, 3) for e in ex]} max/mean {max(ex) / mean:.4f}", flush=True)
