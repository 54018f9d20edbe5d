"""GPU: the single-process multi-GPU group (shtc_group, the reference's in-process workers of
distributed_synthesis / distributed_analysis, distribution.cpp:300-490).  W worker contexts run
on the devices present (all on device 0 here); the Delta exchange is the fused one (producer
kernels store straight into the consumers' buffers, consumers wait on the producers' events)
or NCCL (grouped send / recv; one distinct device per worker).

Oracle: the reference itself (oracle/_ref) with the same worker count; invariance: the group
equals one context (alm2map bitwise, map2alm to 1e-14)."""
import numpy as np
import pytest

from oracle import ref
from paper_1106_0159_b200 import sht
from paper_1106_0159_b200._lib import SHTC_EUNSUPPORTED, ShtcError

pytestmark = pytest.mark.gpu


def rel_rms(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def as_sht(g):
    return sht.PixelGrid("healpix-ring", g.nside, g.cos_theta, g.n_phi, g.phi_0, g.weight)


@pytest.mark.parametrize("nside,lmax,W,rings", [(16, 40, 1, "blocks"), (16, 40, 2, "blocks"), (32, 64, 3, "blocks"),
                                                 (64, 128, 4, "balanced"), (128, 256, 8, "blocks"),
                                                 (128, 256, 8, "balanced"),
                                                 (1100, 64, 2, "balanced")])  # split 8192-point Bluestein class
def test_group_matches_reference_and_one_context(nside, lmax, W, rings):
    g = ref.healpix_grid(nside)
    sg = as_sht(g)
    alm = ref.random_alm(lmax, lmax, 12345)
    want, _ = ref.distributed_synthesis(alm, lmax, lmax, g, n_workers=W, n_threads=4, pairing=True)
    want_alm, _ = ref.distributed_analysis(want, lmax, lmax, g, n_workers=W, n_threads=4, pairing=True)
    one = sht.Context(0)
    one.set_grid(sg)
    one.set_band(lmax, lmax)
    one_map = one.alm2map(alm)
    one_alm = one.map2alm(want)
    grp = sht.Group(W)
    grp.set_grid(sg)
    lay = sht.WorkerLayout.create(sg, lmax, W, rings=rings)
    grp.set_layout(lmax, lmax, lay.m_sets, lay.ring_sets)
    got, t = grp.alm2map(alm, timing=True)
    assert np.array_equal(got, one_map)
    assert rel_rms(got, want) <= 1e-12
    back, t2 = grp.map2alm(want, timing=True)
    assert rel_rms(back, one_alm) <= 1e-14
    assert rel_rms(back, want_alm) <= 1e-12
    for tt in (t, t2):
        assert tt["legendre_ms"] > 0 and tt["fft_ms"] > 0 and tt["total_ms"] > 0
        assert tt["nominal_steps"] == (lmax + 1) * (lmax + 2) // 2 * ((g.n_rings + 1) // 2)
        if W > 1:
            assert tt["exchange_bytes"] > 0
    # repeated calls in one direction: the next call's peer stores wait for every worker's
    # previous consumer stage (write-after-read)
    for _ in range(3):
        assert np.array_equal(grp.alm2map(alm), one_map)
    first = grp.map2alm(want)
    for _ in range(2):
        assert np.array_equal(grp.map2alm(want), first)
    grp.close()
    one.close()


def test_group_device_buffers_and_pinned_host():
    """shtc_group_*_dev: per-worker full-size device buffers (each worker reads its orders /
    writes its rings), and page-locked host buffers (no staging)."""
    import torch

    nside, lmax, W = 64, 128, 4
    sg = sht.build_healpix_grid(nside)
    alm = sht.gaussian_alm(lmax, lmax, 7)
    grp = sht.Group(W)
    grp.set_grid(sg)
    lay = sht.WorkerLayout.create(sg, lmax, W)
    grp.set_layout(lmax, lmax, lay.m_sets, lay.ring_sets)
    want_map = grp.alm2map(alm)
    want_alm = grp.map2alm(want_map)
    dev = torch.device("cuda", 0)
    a = [torch.from_numpy(alm.view(np.float64).copy()).to(dev) for _ in range(W)]
    m = [torch.zeros(sg.n_pix, dtype=torch.float64, device=dev) for _ in range(W)]
    torch.cuda.synchronize()
    grp.alm2map_dev([x.data_ptr() for x in a], [x.data_ptr() for x in m])
    got = np.zeros(sg.n_pix)
    off = np.asarray(sg.pixel_offset)
    nphi = np.asarray(sg.n_phi)
    for w in range(W):
        mw = m[w].cpu().numpy()
        for r in lay.ring_sets[w]:
            got[off[r]:off[r] + nphi[r]] = mw[off[r]:off[r] + nphi[r]]
    assert np.array_equal(got, want_map)
    out = [torch.zeros_like(a[0]) for _ in range(W)]
    for w in range(W):
        m[w].copy_(torch.from_numpy(want_map).to(dev))
    torch.cuda.synchronize()
    grp.map2alm_dev([x.data_ptr() for x in m], [x.data_ptr() for x in out])
    back = np.zeros_like(alm)
    for w in range(W):
        ow = out[w].cpu().numpy().view(np.complex128)
        for mm in lay.m_sets[w]:
            o = sht.alm_offset(mm, lmax)
            back[o:o + lmax - mm + 1] = ow[o:o + lmax - mm + 1]
    assert np.array_equal(back, want_alm)
    alm_pin = torch.from_numpy(alm.view(np.float64).copy()).pin_memory()
    map_pin = torch.empty(sg.n_pix, dtype=torch.float64).pin_memory()
    grp.alm2map(alm_pin.numpy().view(np.complex128), out=map_pin.numpy())
    assert np.array_equal(map_pin.numpy(), want_map)
    grp.close()


def test_group_nccl_exchange():
    """NCCL exchange (ncclCommInitAll + grouped ncclSend / ncclRecv): one worker per device;
    workers sharing a device are refused (NCCL has one rank per device)."""
    n_dev = sht.device_count()
    nside, lmax = 32, 64
    sg = sht.build_healpix_grid(nside)
    alm = sht.random_alm(lmax, lmax, 3)
    one = sht.Context(0)
    one.set_grid(sg)
    one.set_band(lmax, lmax)
    want = one.alm2map(alm)
    want_alm = one.map2alm(want)
    for W in sorted({1, min(2, n_dev), min(4, n_dev)}):
        grp = sht.Group(W, devices=list(range(W)), exchange="nccl")
        grp.set_grid(sg)
        lay = sht.WorkerLayout.create(sg, lmax, W)
        grp.set_layout(lmax, lmax, lay.m_sets, lay.ring_sets)
        got, t = grp.alm2map(alm, timing=True)
        assert np.array_equal(got, want)
        back = grp.map2alm(want)
        assert rel_rms(back, want_alm) <= 1e-14
        grp.close()
    if n_dev == 1:
        with pytest.raises(ShtcError) as ei:
            sht.Group(2, devices=[0, 0], exchange="nccl")
        assert ei.value.code == SHTC_EUNSUPPORTED


def test_group_layout_errors():
    sg = sht.build_healpix_grid(8)
    grp = sht.Group(2)
    grp.set_grid(sg)
    with pytest.raises(ValueError):
        grp.set_layout(16, 16, [[0, 1, 2], [3, 4]], [list(range(sg.n_rings)), []])  # worker 1: no ring
    lay = sht.WorkerLayout.create(sg, 16, 2)
    grp.set_layout(16, 16, lay.m_sets, lay.ring_sets)
    with pytest.raises(ValueError):
        grp.alm2map(np.zeros(5, np.complex128))
    grp.close()
