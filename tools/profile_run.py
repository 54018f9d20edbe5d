"""One device-resident alm2map + map2alm at a given HEALPix config (for ncu captures)."""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1106_0159_b200 import sht
p = argparse.ArgumentParser()
p.add_argument("--nside", type=int, default=1024)
p.add_argument("--lmax", type=int, default=2048)
p.add_argument("--iters", type=int, default=1)
a = p.parse_args()
g = sht.build_healpix_grid(a.nside)
ctx = sht.Context(0)
ctx.set_grid(g); ctx.set_band(a.lmax, a.lmax); ctx.plan()
alm = torch.from_numpy(sht.gaussian_alm(a.lmax, a.lmax, 12345).view(np.float64)).cuda()
mp = torch.empty(g.n_pix, dtype=torch.float64, device="cuda")
alm2 = torch.empty_like(alm)
torch.cuda.synchronize()
for _ in range(a.iters):
    t1 = ctx.alm2map_dev(alm.data_ptr(), mp.data_ptr(), timing=True)
    t2 = ctx.map2alm_dev(mp.data_ptr(), alm2.data_ptr(), timing=True)
    print("alm2map", t1, "\nmap2alm", t2, flush=True)
