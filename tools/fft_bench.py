"""C4 ring-stage timing (ms) of the library SHTC_VARIANT_LIB points at (default: the shipped one)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1106_0159_b200 import sht
nside = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
lmax = 2 * nside
g = sht.build_healpix_grid(nside)
ctx = sht.Context(0)
ctx.set_grid(g); ctx.set_band(lmax, lmax); ctx.plan()
alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 12345).view(np.float64)).cuda()
mp = torch.empty(g.n_pix, dtype=torch.float64, device="cuda")
alm2 = torch.empty_like(alm)
a, m = [], []
for _ in range(6):
    a.append(ctx.alm2map_dev(alm.data_ptr(), mp.data_ptr(), timing=True)["fft_ms"])
    m.append(ctx.map2alm_dev(mp.data_ptr(), alm2.data_ptr(), timing=True)["fft_ms"])
print(f"{os.environ.get('SHTC_VARIANT_LIB', 'default')}: synth_fft={min(a[1:]):.3f} anal_fft={min(m[1:]):.3f}", flush=True)
