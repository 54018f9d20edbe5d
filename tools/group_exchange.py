"""Single-process group (shtc_group, fused peer-store exchange) on the devices at hand: W
workers (all on device 0 when there is one GPU), device-resident a_lm / map, per-stage times
from the group's own events.  SHTC_GROUP_RING_MAJOR=1 selects the ring-major synthesis
blocks (the comparison layout for the order-major default).

    python tools/group_exchange.py --nside 1024 --lmax 2048 --workers 2 4 8
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import sht


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nside", type=int, default=1024)
    ap.add_argument("--lmax", type=int, default=2048)
    ap.add_argument("--workers", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n_dev = sht.device_count()
    grid = sht.build_healpix_grid(a.nside)
    lmax = a.lmax
    alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 12345).view(np.float64)).cuda()
    for W in a.workers:
        devs = [w % n_dev for w in range(W)]
        grp = sht.Group(W, devices=devs)
        grp.set_grid(grid)
        lay = sht.WorkerLayout.create(grid, lmax, W)
        grp.set_layout(lmax, lmax, lay.m_sets, lay.ring_sets)
        maps = [torch.zeros(grid.n_pix, dtype=torch.float64, device=f"cuda:{d}") for d in devs]
        alms = [alm.to(f"cuda:{d}") for d in devs]
        outs = [torch.zeros_like(x) for x in alms]
        rec = {"a2m": [], "m2a": []}
        for _ in range(a.reps):
            rec["a2m"].append(grp.alm2map_dev([x.data_ptr() for x in alms], [m.data_ptr() for m in maps]))
            rec["m2a"].append(grp.map2alm_dev([m.data_ptr() for m in maps], [x.data_ptr() for x in outs]))
        best = {k: min(v, key=lambda t: t["total_ms"]) for k, v in rec.items()}
        line = {"W": W, "devices": devs, "nside": a.nside, "lmax": lmax,
                "layout": "ring-major" if os.environ.get("SHTC_GROUP_RING_MAJOR") == "1" else "order-major",
                **{f"{k}_{f}": best[k][f] for k in best for f in ("legendre_ms", "fft_ms", "exchange_ms", "total_ms",
                                                                      "exchange_bytes")}}
        print(json.dumps(line), flush=True)
        grp.close()


if __name__ == "__main__":
    main()
