"""Parity spot-check + C4 Legendre timing of the library SHTC_VARIANT_LIB points at.

    SHTC_VARIANT_LIB=paper_1106_0159_b200/_build/var_x/libshtc.so python tools/variant_bench.py
"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from oracle import ref
from paper_1106_0159_b200 import sht

def rr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

ctx = sht.Context(0)
errs = []
for nside, lmax in ((4, 12), (32, 64), (128, 256)):
    g = ref.healpix_grid(nside)
    alm = ref.random_alm(lmax, lmax, 12345)
    want, _ = ref.synthesis(alm, lmax, lmax, g, pairing=True)
    ctx.set_grid(sht.PixelGrid("h", nside, g.cos_theta, g.n_phi, g.phi_0, g.weight)); ctx.set_band(lmax, lmax)
    got = ctx.alm2map(alm)
    w2, _ = ref.analysis(want, lmax, lmax, g, pairing=True)
    b = ctx.map2alm(want)
    errs += [rr(got, want), rr(b, w2)]
import torch
g = sht.build_healpix_grid(2048)
ctx.set_grid(g); ctx.set_band(4096, 4096); ctx.plan()
alm = torch.from_numpy(sht.gaussian_alm(4096, 4096, 12345).view(np.float64)).cuda()
mp = torch.empty(g.n_pix, dtype=torch.float64, device="cuda")
alm2 = torch.empty_like(alm)
a, m = [], []
for _ in range(4):
    a.append(ctx.alm2map_dev(alm.data_ptr(), mp.data_ptr(), timing=True)["legendre_ms"])
    m.append(ctx.map2alm_dev(mp.data_ptr(), alm2.data_ptr(), timing=True)["legendre_ms"])
st = ctx.plan_stats()
print(f"{os.environ.get('SHTC_VARIANT_LIB', 'default')}: max_err={max(errs):.2e} a2m={min(a[1:]):.3f} m2a={min(m[1:]):.3f} executed={st}", flush=True)
