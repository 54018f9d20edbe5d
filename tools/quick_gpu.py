import sys, time; sys.path.insert(0,'.')
import numpy as np
from oracle import ref
from paper_1106_0159_b200 import sht
def rr(a,b): return float(np.linalg.norm(a-b)/np.linalg.norm(b)), float(np.abs(a-b).max()/np.abs(b).max())
ctx=sht.Context(0)
print(sht.device_info(0), sht.measure_fp64_peak(0))
for nside,lmax in ((1,2),(2,5),(4,12),(8,20),(32,64),(128,256)):
    g=ref.healpix_grid(nside); alm=ref.random_alm(lmax,lmax,12345)
    want,_=ref.synthesis(alm,lmax,lmax,g,pairing=True)
    ctx.set_grid(sht.PixelGrid("h",nside,g.cos_theta,g.n_phi,g.phi_0,g.weight)); ctx.set_band(lmax,lmax)
    got=ctx.alm2map(alm)
    w2,_=ref.analysis(want,lmax,lmax,g,pairing=True); b=ctx.map2alm(want)
    print(nside,lmax,"synth",rr(got,want),"anal",rr(b,w2), ctx.plan_stats(), flush=True)
for nside,lmax in ((1024,2048),(2048,4096)):
    g=ref.healpix_grid(nside); alm=sht.gaussian_alm(lmax,lmax,12345)
    ctx.set_grid(sht.PixelGrid("h",nside,g.cos_theta,g.n_phi,g.phi_0,g.weight)); ctx.set_band(lmax,lmax)
    t0=time.time(); pm=ctx.plan(); print("plan ms",pm,"wall",time.time()-t0, ctx.plan_stats(), flush=True)
    for it in range(3):
        mp,t=ctx.alm2map(alm,timing=True); print("alm2map",t, flush=True)
        a2,t=ctx.map2alm(mp,timing=True); print("map2alm",t, flush=True)
