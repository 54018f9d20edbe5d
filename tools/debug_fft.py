import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import ref
from paper_1106_0159_b200 import sht
ctx=sht.Context(0)
lmax=40
alm=ref.random_alm(lmax,lmax,3)
for nphi in [4,6,8,9,10,26,34,128,254,256,258,260,300,400,510,512,600,1000,1022,1024,1030,2046,2048,4094,4096,5000,8188,8192,8190,7,101,999,2049]:
    g=ref.gl_grid(5,nphi)
    want,_=ref.synthesis(alm,lmax,lmax,g,pairing=True)
    ctx.set_grid(sht.PixelGrid("g",0,g.cos_theta,g.n_phi,g.phi_0,g.weight)); ctx.set_band(lmax,lmax)
    got=ctx.alm2map(alm)
    e1=np.abs(got-want).max()/np.abs(want).max()
    w2,_=ref.analysis(want,lmax,lmax,g,pairing=True); b=ctx.map2alm(want)
    e2=np.abs(b-w2).max()/np.abs(w2).max()
    N=nphi//2 if nphi%2==0 else nphi
    print(nphi,"N",N,"synth",e1,"anal",e2, flush=True)
