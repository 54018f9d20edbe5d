"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family of the library through the C ABI, with host buffers only (no torch), checked against
the oracle so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck --error-exitcode 3 python tools/sanitize_run.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np

from oracle import ref
from paper_1106_0159_b200 import sht


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


ctx = sht.Context(0)
worst = 0.0
# HEALPix (mirror pairs, power-of-two and Bluestein ring classes, aliasing caps) and a
# Gauss-Legendre grid with odd n_phi (generic mixed-radix class)
# rings of 6002 samples (N = 3001: 8192-point Bluestein, the split two-group kernel) and of
# 8194 (N = 4097: not 7-smooth, 16384-point 2-CTA cluster class)
cases = [(ref.healpix_grid(64), 128), (ref.healpix_grid(8), 40), (ref.gl_grid(17, 35), 16),
         (ref.gl_grid(6, 6002), 5), (ref.gl_grid(4, 8194), 3)]
for g, lmax in cases:
    alm = ref.random_alm(lmax, lmax, 99)
    want, _ = ref.synthesis(alm, lmax, lmax, g, pairing=True)
    back_want, _ = ref.analysis(want, lmax, lmax, g, pairing=True)
    ctx.set_grid(sht.PixelGrid("x", g.nside, g.cos_theta, g.n_phi, g.phi_0, g.weight))
    ctx.set_band(lmax, lmax)
    got = ctx.alm2map(alm)  # pipelined host path: band launches, finalize, copies
    back = ctx.map2alm(want)
    worst = max(worst, rel(got, want), rel(back, back_want))
# Legendre-stage operators (unpaired streams, accumulate into a_lm)
lmax = 24
x = np.cos(np.linspace(0.05, 3.1, 11))
ms = [0, 3, 7, 24]
alm = ref.random_alm(lmax, lmax, 5)
want, _ = ref.compute_delta_a(alm, lmax, lmax, x, ms)
got, _ = ctx.delta_a(alm, lmax, lmax, x, ms)
worst = max(worst, rel(got, want))
ctx.close()
print(f"sanitize_run ok: worst rel {worst:.2e}")
assert worst < 1e-12, worst
