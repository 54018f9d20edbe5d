"""GPU parity at the north-star configs: C4 (nside 2048, lmax = mmax = 4096) and C5 (nside 4096,
lmax = mmax = 8192), whole alm2map and map2alm through the C ABI host-buffer entry points
against the reference (oracle/_ref: the unmodified reference sources compiled here, on all
host threads, PairPolicy::mirror -- transforms.cpp:402-485 via distributed_synthesis /
distributed_analysis, distribution.cpp:300-490).

Inputs (SURVEY.md §8c/§8d protocol):
  * random_alm (uniform re/im, seed 12345), the parity input;
  * gaussian_alm (N(0,1) re/im, seed 12345), the bench's throughput input;
  * an i.i.d. N(0,1) pixel map (seed 2026), a map that is NOT band-limited (map2alm aliasing).
map2alm runs on the oracle's own map (step 4 of the protocol), so the two directions are
checked independently.  Gate: rel-RMS <= 1e-10 (north star), worst case reported and bounded.
Each test records its numbers under gpurun_out/parity/ (one JSON per test).
"""
import json
import os
import time
from pathlib import Path

import numpy as np
import pytest

from oracle import ref
from paper_1106_0159_b200 import sht

pytestmark = pytest.mark.gpu

RMS_TOL = 1e-10      # north star: map and a_lm rel-RMS
WORST_TOL = 1e-9     # max|diff| / max|ref|, reported; the recurrence's own conditioning at x -> 1
THREADS = os.cpu_count() or 1
OUT = Path(__file__).resolve().parents[1] / "gpurun_out" / "parity"


def rel_rms(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def worst(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def record(name, **kw):
    OUT.mkdir(parents=True, exist_ok=True)
    rec = {"test": name, "ref_threads": THREADS, "gate_rel_rms": RMS_TOL, **kw}
    (OUT / f"{name}.json").write_text(json.dumps(rec) + "\n")
    print(json.dumps(rec))


_GRIDS = {}


def grids(nside):
    if nside not in _GRIDS:
        g = ref.healpix_grid(nside)
        _GRIDS[nside] = (g, sht.PixelGrid("healpix-ring", nside, g.cos_theta, g.n_phi, g.phi_0, g.weight))
    return _GRIDS[nside]


@pytest.fixture(scope="module")
def ctx():
    c = sht.Context(0)
    yield c
    c.close()


def _bind(ctx, nside, lmax):
    _, sg = grids(nside)
    if getattr(ctx, "_cfg", None) != (nside, lmax):
        ctx.set_grid(sg, mirror=True)
        ctx.set_band(lmax, lmax)
        ctx._cfg = (nside, lmax)


def _both_directions(ctx, name, nside, lmax, alm, what):
    g, _ = grids(nside)
    _bind(ctx, nside, lmax)
    t0 = time.perf_counter()
    want, _ = ref.distributed_synthesis(alm, lmax, lmax, g, n_workers=1, n_threads=THREADS, pairing=True)
    t_ref1 = time.perf_counter() - t0
    got = ctx.alm2map(alm)
    r1, w1 = rel_rms(got, want), worst(got, want)
    t0 = time.perf_counter()
    back_ref, _ = ref.distributed_analysis(want, lmax, lmax, g, n_workers=1, n_threads=THREADS, pairing=True)
    t_ref2 = time.perf_counter() - t0
    back = ctx.map2alm(want)
    r2, w2 = rel_rms(back, back_ref), worst(back, back_ref)
    record(name, config=f"HEALPix nside={nside} lmax=mmax={lmax}", input=what,
           alm2map={"rel_rms": r1, "worst": w1, "ref_s": t_ref1},
           map2alm={"rel_rms": r2, "worst": w2, "ref_s": t_ref2, "input": "the oracle's alm2map output"})
    assert r1 <= RMS_TOL and w1 <= WORST_TOL, (r1, w1)
    assert r2 <= RMS_TOL and w2 <= WORST_TOL, (r2, w2)


def _iid_map(ctx, name, nside, lmax):
    g, sg = grids(nside)
    _bind(ctx, nside, lmax)
    mp = sht.gaussian_map(sg.n_pix, 2026)
    t0 = time.perf_counter()
    want, _ = ref.distributed_analysis(mp, lmax, lmax, g, n_workers=1, n_threads=THREADS, pairing=True)
    t_ref = time.perf_counter() - t0
    got = ctx.map2alm(mp)
    r, w = rel_rms(got, want), worst(got, want)
    record(name, config=f"HEALPix nside={nside} lmax=mmax={lmax}",
           input="i.i.d. N(0,1) pixel map, seed 2026 (not band-limited)",
           map2alm={"rel_rms": r, "worst": w, "ref_s": t_ref})
    assert r <= RMS_TOL and w <= WORST_TOL, (r, w)


def test_c2_map2alm_iid_map(ctx):
    _iid_map(ctx, "c2_map2alm_iid_map", 1024, 2048)


def test_c4_uniform_alm_alm2map_map2alm(ctx):
    """C4 with the reference's random_alm (uniform re/im, Im a_l0 = 0), seed 12345."""
    lmax = 4096
    _both_directions(ctx, "c4_uniform_alm", 2048, lmax, ref.random_alm(lmax, lmax, 12345),
                     "random_alm seed 12345 (uniform re/im)")


def test_c4_gaussian_alm_alm2map_map2alm(ctx):
    """C4 with the bench's Gaussian a_lm (N(0,1) re/im by Box-Muller), seed 12345."""
    lmax = 4096
    _both_directions(ctx, "c4_gaussian_alm", 2048, lmax, sht.gaussian_alm(lmax, lmax, 12345),
                     "gaussian_alm seed 12345 (N(0,1) re/im)")


def test_c4_map2alm_iid_map(ctx):
    _iid_map(ctx, "c4_map2alm_iid_map", 2048, 4096)


def test_c4_device_path_matches_host_path(ctx):
    """The device-resident entry points (what bench.py's `value` times) give the host-buffer
    results at C4: alm2map bitwise, map2alm to 1e-14 (per-band partial-sum grouping)."""
    import torch

    lmax = 4096
    _bind(ctx, 2048, lmax)
    _, sg = grids(2048)
    alm = sht.gaussian_alm(lmax, lmax, 12345)
    dev = torch.device("cuda:0")
    ad = torch.from_numpy(alm.view(np.float64).copy()).to(dev)
    md = torch.empty(sg.n_pix, dtype=torch.float64, device=dev)
    bd = torch.empty_like(ad)
    torch.cuda.synchronize()
    ctx.alm2map_dev(ad.data_ptr(), md.data_ptr())
    ctx.map2alm_dev(md.data_ptr(), bd.data_ptr())
    torch.cuda.synchronize()
    mp = ctx.alm2map(alm)
    assert np.array_equal(md.cpu().numpy(), mp)
    back = ctx.map2alm(mp)
    assert rel_rms(bd.cpu().numpy().view(np.complex128), back) <= 1e-14


def test_c5_uniform_alm_alm2map_map2alm(ctx):
    """C5 (nside 4096, lmax = mmax = 8192): the deepest underflow ladder (k ~ -200 at the
    polar rings) and the 2-CTA 16384-point Bluestein ring class, whole transforms."""
    lmax = 8192
    _both_directions(ctx, "c5_uniform_alm", 4096, lmax, ref.random_alm(lmax, lmax, 12345),
                     "random_alm seed 12345 (uniform re/im)")


def test_c5_map2alm_iid_map(ctx):
    _iid_map(ctx, "c5_map2alm_iid_map", 4096, 8192)
