"""Parity of the GPU transforms against the reference (oracle/_ref) at a large config, on the
same a_lm: rel-RMS and worst-case of the map (alm2map) and of a_lm (map2alm of the reference's
map).  Writes one JSON line (committed under profiles/ as evidence).

    python tools/parity_large.py --nside 4096 --lmax 8192      # C5
"""
import argparse, json, os, sys, time
sys.path.insert(0, '.')
import numpy as np
from oracle import ref
from paper_1106_0159_b200 import sht

ap = argparse.ArgumentParser()
ap.add_argument("--nside", type=int, default=4096)
ap.add_argument("--lmax", type=int, default=8192)
ap.add_argument("--seed", type=int, default=12345)
a = ap.parse_args()
nth = os.cpu_count() or 1
g = ref.healpix_grid(a.nside)
alm = ref.random_alm(a.lmax, a.lmax, a.seed)
ctx = sht.Context(0)
ctx.set_grid(sht.PixelGrid("h", a.nside, g.cos_theta, g.n_phi, g.phi_0, g.weight))
ctx.set_band(a.lmax, a.lmax)
t0 = time.perf_counter(); got = ctx.alm2map(alm); t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
want, _ = ref.distributed_synthesis(alm, a.lmax, a.lmax, g, n_workers=1, n_threads=nth, pairing=True)
t_ref = time.perf_counter() - t0
t0 = time.perf_counter(); back = ctx.map2alm(want); t_gpu2 = time.perf_counter() - t0
t0 = time.perf_counter()
back_ref, _ = ref.distributed_analysis(want, a.lmax, a.lmax, g, n_workers=1, n_threads=nth, pairing=True)
t_ref2 = time.perf_counter() - t0


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y)), float(np.max(np.abs(x - y)) / np.max(np.abs(y)))


r1, w1 = rel(got, want)
r2, w2 = rel(back, back_ref)
print(json.dumps({"config": f"HEALPix nside={a.nside} lmax=mmax={a.lmax}", "seed": a.seed,
                  "alm2map": {"rel_rms": r1, "worst": w1, "gpu_s_host_api": t_gpu, "ref_s": t_ref},
                  "map2alm": {"rel_rms": r2, "worst": w2, "gpu_s_host_api": t_gpu2, "ref_s": t_ref2},
                  "ref_threads": nth, "gate": "rel_rms <= 1e-10 (north star)"}), flush=True)
