"""GPU: the multi-GPU stage path (Legendre -> packed all-to-all buffers -> ring stage) run for
W workers on one device, the all-to-all emulated by block copies exactly as NCCL moves them.
Must be bitwise equal to the single-worker transform (distribution.cpp's invariance,
test_distribution.cpp:256-311)."""
import numpy as np
import pytest
import torch

from paper_1106_0159_b200 import sht

pytestmark = pytest.mark.gpu


def alltoall(sends, send_counts, recv_counts, W):
    """sends[j]: flat complex buffer of worker j, blocks for destinations 0..W-1."""
    out = []
    for i in range(W):
        parts = []
        for j in range(W):
            off = sum(send_counts[j][:i])
            parts.append(sends[j][2 * off: 2 * (off + send_counts[j][i])])
        out.append(torch.cat(parts))
        assert out[-1].numel() == 2 * sum(recv_counts[i])
    return out


@pytest.mark.parametrize("nside,lmax,W,rings", [(8, 16, 1, "blocks"), (8, 16, 2, "blocks"), (16, 40, 3, "blocks"),
                                                 (64, 128, 4, "blocks"), (128, 256, 8, "blocks"),
                                                 (256, 512, 1, "blocks"), (64, 128, 4, "balanced"),
                                                 (128, 256, 8, "balanced"), (16, 40, 3, "interleaved"),
                                                 # polar caps of 4100..4396 samples: the split 8192-point
                                                 # Bluestein class through the exchange layouts
                                                 (1100, 64, 4, "balanced")])
@pytest.mark.parametrize("order_major", [True, False])
def test_stage_path_matches_single_worker(nside, lmax, W, rings, order_major):
    dev = torch.device("cuda", 0)
    grid = sht.build_healpix_grid(nside)
    alm_h = sht.random_alm(lmax, lmax, 99)
    alm = torch.from_numpy(alm_h.view(np.float64)).to(dev)
    single = sht.Context(0)
    single.set_grid(grid)
    single.set_band(lmax, lmax)
    want_map = torch.from_numpy(single.alm2map(alm_h)).to(dev)
    want_alm = single.map2alm(want_map.cpu().numpy())

    layout = sht.WorkerLayout.create(grid, lmax, W, rings=rings)
    ctxs, metas = [], []
    for w in range(W):
        c = sht.Context(0)
        c.set_grid(grid)
        c.set_band(lmax, lmax, layout.m_sets[w])
        meta = sht.exchange_layout(layout, w)
        row_off, send_c, recv_c, ring_list, m_base, m_stride = meta
        c.set_exchange_layout(row_off, ring_list, m_base, m_stride)
        if order_major:  # alm2map blocks order-major (the fused / NCCL default)
            c.set_exchange_layout_synthesis(*sht.exchange_layout_synthesis(layout, w))
        ctxs.append(c)
        metas.append(meta)
    send_counts = [m[1] for m in metas]
    recv_counts = [m[2] for m in metas]
    # alm2map: Legendre into the send buffers
    sends = []
    for w in range(W):
        buf = torch.empty(2 * sum(send_counts[w]), dtype=torch.float64, device=dev)
        ctxs[w].legendre_alm2map_dev(alm.data_ptr(), buf.data_ptr())
        sends.append(buf)
    torch.cuda.synchronize()
    recvs = alltoall(sends, send_counts, recv_counts, W)
    mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
    for w in range(W):
        ctxs[w].ring_synthesis_dev(recvs[w].data_ptr(), mp.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(mp, want_map)
    # map2alm: ring stage into receive-shaped blocks, reverse all-to-all, Legendre per worker
    blocks = []
    for w in range(W):
        buf = torch.empty(2 * sum(recv_counts[w]), dtype=torch.float64, device=dev)
        ctxs[w].ring_analysis_dev(want_map.data_ptr(), buf.data_ptr())
        blocks.append(buf)
    torch.cuda.synchronize()
    back = alltoall(blocks, recv_counts, send_counts, W)
    out = torch.zeros(2 * sht.alm_count(lmax, lmax), dtype=torch.float64, device=dev)
    for w in range(W):
        ctxs[w].legendre_map2alm_dev(back[w].data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.complex128)
    assert np.array_equal(got, want_alm)


def test_copy_orders_moves_exactly_the_worker_orders():
    """shtc_copy_orders: a worker's order segments between full host / device a_lm triangles
    (the multi-rank e2e path); other orders untouched."""
    dev = torch.device("cuda", 0)
    lmax = 40
    grid = sht.build_healpix_grid(16)
    layout = sht.WorkerLayout.create(grid, lmax, 3)
    ms = layout.m_sets[1]
    c = sht.Context(0)
    c.set_grid(grid)
    c.set_band(lmax, lmax, ms)
    alm_h = sht.random_alm(lmax, lmax, 5)
    host = torch.from_numpy(alm_h.view(np.float64).copy()).pin_memory()
    d = torch.full((host.numel(),), -7.0, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    c.copy_orders(host.data_ptr(), d.data_ptr(), True)
    torch.cuda.synchronize()
    back = torch.full_like(host, 3.0).pin_memory()
    c.copy_orders(d.data_ptr(), back.data_ptr(), False)
    torch.cuda.synchronize()
    got_d = d.cpu().numpy().view(np.complex128)
    got_b = back.numpy().view(np.complex128)
    mine = np.zeros(alm_h.size, bool)
    for m in ms:
        o = sht.alm_offset(m, lmax)
        mine[o:o + lmax - m + 1] = True
    assert np.array_equal(got_d[mine], alm_h[mine]) and np.all(got_d[~mine] == -7.0 - 7.0j)
    assert np.array_equal(got_b[mine], alm_h[mine]) and np.all(got_b[~mine] == 3.0 + 3.0j)
    c.close()
