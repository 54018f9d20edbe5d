"""GPU parity of the ring Fourier stage over every FFT size class (ringfft.cu).

One grid per case holds rings of many different lengths, so a single alm2map / map2alm touches
the generic mixed-radix classes (tiny, odd and 7-smooth rings), the power-of-two engine's direct
classes (N = 256 ... 8192), its Bluestein classes (buffers 256 ... 8192) and the 2-CTA cluster
class (Bluestein buffers of 16384), with phi_0 = 0 and
phi_0 != 0 rings and with orders above n/2 (aliasing folds).  Oracle: the reference's
synthesis / analysis (fourier.cpp:10-56 + fft.cpp) on the same grid and a_lm.
"""
import os

import numpy as np
import pytest

from oracle import ref
from paper_1106_0159_b200 import sht

pytestmark = pytest.mark.gpu

# ring lengths -> (complex length N, engine class) at the planner's rules
NPHI = [
    4, 6, 7, 34, 101, 999,      # generic: tiny, odd (full-length complex FFT), small smooth
    130, 254,                   # Bluestein, buffer 256
    256,                        # direct N = 128 (generic class)
    512, 1024,                  # direct N = 256, 512 (power-of-two engine)
    1000, 1030,                 # smooth N = 500 (generic), Bluestein N = 515 (buffer 2048)
    2048, 2052,                 # direct N = 1024, Bluestein N = 1026 (buffer 4096)
    4096, 4100,                 # direct N = 2048, Bluestein N = 2050 (buffer 8192)
    6000,                       # 7-smooth N = 3000 > 1024: Bluestein buffer 8192
    8188, 8192,                 # Bluestein N = 4094 (8192), direct N = 4096
    16384,                      # direct N = 8192
    8200, 12000, 16380,         # Bluestein N = 4100, 6000 (7-smooth), 8190: 16384-point, 2-CTA cluster
    4099, 5005, 8191, 8193,     # odd, beyond the generic classes: pruned one-sided Bluestein, cluster
]


def mixed_grid(nphi, phase):
    nr = 2 * len(nphi)
    x, w = ref.gl_nodes(nr)
    x = np.asarray(x)[::-1].copy()
    w = np.asarray(w)[::-1].copy()
    n = np.array(list(nphi) + list(nphi)[::-1], dtype=np.int32)  # mirror pairs share a length
    phi0 = np.where(np.arange(nr) % 2 == 1, phase * np.pi / n, 0.0) if phase else np.zeros(nr)
    weight = w * 2.0 * np.pi / n
    return ref.Grid(1, 0, x, n, phi0, weight)


def rel_max(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("lmax,phase", [(40, 0.0), (40, 0.5), (700, 0.5), (4200, 0.25)])
def test_ring_classes_match_reference(gpu_ctx, lmax, phase):
    nphi = NPHI if lmax < 4000 else [4, 130, 1030, 4100, 8188, 8192, 16384, 8200, 16380, 4099, 8193, 12001]
    g = mixed_grid(nphi, phase)
    alm = ref.random_alm(lmax, lmax, 4242)
    want, _ = ref.synthesis(alm, lmax, lmax, g, pairing=True)
    gpu_ctx.set_grid(sht.PixelGrid("x", 0, g.cos_theta, g.n_phi, g.phi_0, g.weight))
    gpu_ctx.set_band(lmax, lmax)
    got = gpu_ctx.alm2map(alm)
    off = np.concatenate([[0], np.cumsum(g.n_phi)])
    for r in range(len(g.n_phi)):
        a, b = got[off[r]:off[r + 1]], want[off[r]:off[r + 1]]
        assert rel_max(a, b) < 1e-12, (r, int(g.n_phi[r]), rel_max(a, b))
    back_want, _ = ref.analysis(want, lmax, lmax, g, pairing=True)
    back = gpu_ctx.map2alm(want)
    assert rel_max(back, back_want) < 1e-12, rel_max(back, back_want)


@pytest.mark.parametrize("nphi,mmax", [(32768, 8), (65540, 8), (16001, 1000), (9001, 8000)])
def test_unsupported_ring_lengths_fail_loudly(gpu_ctx, nphi, mmax):
    """Ring lengths beyond the size classes (direct N = 16384, i.e. n_phi = 32768 / HEALPix
    nside >= 8192 belt rings; Bluestein buffers above 16384, half-length or, for odd n_phi, the
    pruned n_phi + min(n_phi, mmax + 1) - 1) are refused with SHTC_EUNSUPPORTED at plan time,
    never computed wrongly."""
    from paper_1106_0159_b200._lib import SHTC_EUNSUPPORTED, ShtcError
    g = mixed_grid([16, nphi], 0.0)
    gpu_ctx.set_grid(sht.PixelGrid("x", 0, g.cos_theta, g.n_phi, g.phi_0, g.weight))
    gpu_ctx.set_band(mmax, mmax)
    with pytest.raises(ShtcError) as ei:
        gpu_ctx.alm2map(ref.random_alm(mmax, mmax, 1))
    assert ei.value.code == SHTC_EUNSUPPORTED
    assert "ring length" in str(ei.value)


def test_gauss_legendre_2lmax_plus_1_at_lmax_4096(gpu_ctx):
    """GL(4097, 8193) at lmax = mmax = 4096 -- the classic n_phi = 2 lmax + 1 choice
    (acceptance.cpp's GL(256, 513) at C4's band): odd rings of 8193 samples on the pruned
    one-sided Bluestein class, against the reference on all host threads."""
    lmax = 4096
    g = ref.gl_grid(lmax + 1, 2 * lmax + 1)
    alm = ref.random_alm(lmax, lmax, 2026)
    threads = os.cpu_count() or 1
    want, _ = ref.distributed_synthesis(alm, lmax, lmax, g, n_workers=1, n_threads=threads, pairing=True)
    gpu_ctx.set_grid(sht.PixelGrid("x", 0, g.cos_theta, g.n_phi, g.phi_0, g.weight))
    gpu_ctx.set_band(lmax, lmax)
    got = gpu_ctx.alm2map(alm)
    e_map = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    back_want, _ = ref.distributed_analysis(want, lmax, lmax, g, n_workers=1, n_threads=threads, pairing=True)
    back = gpu_ctx.map2alm(want)
    e_alm = float(np.linalg.norm(back - back_want) / np.linalg.norm(back_want))
    assert e_map <= 1e-10 and e_alm <= 1e-10, (e_map, e_alm)
