import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import ref
from paper_1106_0159_b200 import sht
ctx=sht.Context(0)
def run(nlat, lmax, label, xs=None):
    if xs is None: xs=np.linspace(0.999,0.001,nlat)
    alm=ref.random_alm(lmax,lmax,3)
    ms=np.arange(lmax+1)
    want,_=ref.compute_delta_a(alm,lmax,lmax,xs,ms)
    got,_=ctx.delta_a(alm,lmax,lmax,xs,ms)
    err=np.abs(got-want)/np.abs(want).max()
    i,j=np.unravel_index(np.nanargmax(np.where(np.isfinite(err),err,1e300)),err.shape)
    print(label,"nlat",nlat,"lmax",lmax,"max err",err[i,j],"at row",i,"m",j,"got",got[i,j],"want",want[i,j], "nbad cols", int(np.sum(np.any(~(err<1e-10),axis=0))), flush=True)
    return err
run(100,64,"1tile 1chunk")
run(100,200,"1tile multichunk")
run(300,64,"3tile 1chunk")
run(300,200,"3tile multichunk")
run(100,60,"1tile 1chunk deep", xs=np.linspace(0.99999,0.001,100))
e=run(128,256,"1tile multichunk deep", xs=np.linspace(0.99999,0.001,128))
print(np.where(~(e<1e-10))[1][:50])
