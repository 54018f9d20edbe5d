"""CPU: host-side code of the product (geometry, inputs, layouts, exchange bookkeeping) and the
multi-worker exchange logic over a world_size-2 gloo group."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

from oracle import sht_oracle as O
from paper_1106_0159_b200 import sht

G = Path(__file__).resolve().parent / "golden"


def test_healpix_geometry_bit_exact():
    k = np.load(G / "kat.npz")
    for ns in (1, 2, 3):
        g = sht.build_healpix_grid(ns)
        want = k[f"hp{ns}"]
        assert np.array_equal(g.cos_theta, want[0])
        assert np.array_equal(g.n_phi.astype(float), want[1])
        assert np.array_equal(g.phi_0, want[2])
    g = sht.build_healpix_grid(2)  # test_grid.cpp:29-45
    assert g.n_rings == 7 and g.n_pix == 48
    assert list(g.n_phi) == [4, 8, 8, 8, 8, 8, 4]
    with pytest.raises(ValueError):
        sht.build_healpix_grid(0)


@pytest.mark.parametrize("name", ["hp4_l12", "hp8_l20", "gl17_l16", "gl10_l9", "gl9_nphi7_l8"])
def test_grids_and_inputs_match_golden(name):
    d = np.load(G / f"transform_{name}.npz")
    n = len(d["cos_theta"])
    if name.startswith("hp"):
        g = sht.build_healpix_grid((n + 1) // 4)
    else:
        g = sht.build_gauss_legendre_grid(n, int(d["n_phi"][0]))
    for f in ("cos_theta", "n_phi", "phi_0", "weight", "pixel_offset"):
        assert np.array_equal(getattr(g, f), d[f]), f
    lmax = int(d["lmax"])
    assert np.array_equal(sht.random_alm(lmax, lmax, int(d["seed"])), d["alm"])


def test_alm_layout():
    assert sht.alm_count(7, 7) == 36 and sht.alm_count(8, 5) == 39
    assert sht.alm_offset(3, 7) == 3 * 8 - 3
    assert sht.alm_index(5, 3, 7) == sht.alm_offset(3, 7) + 2


def test_distribution_layouts():
    # test_distribution.cpp:84-177
    assert sht.assign_m(7, 1) == [list(range(8))]
    assert sht.assign_m(7, 4) == [[0, 7], [1, 6], [2, 5], [3, 4]]
    assert sht.assign_m(7, 2) == [[0, 2, 5, 7], [1, 3, 4, 6]]
    for bad in ((7, 5), (2, 2), (-1, 1), (7, 0)):
        with pytest.raises(ValueError):
            sht.assign_m(*bad)
    hp = sht.build_healpix_grid(2)
    assert sht.assign_rings(hp, 2) == [[0, 1, 5, 6], [2, 3, 4]]
    with pytest.raises(ValueError):
        sht.assign_rings(hp, 4)
    gl = sht.build_gauss_legendre_grid(8, 16)
    assert sht.assign_rings(gl, 4) == [[0, 7], [1, 6], [2, 5], [3, 4]]
    assert sht.thread_partition([0, 2, 5, 7], 2) == [[0, 7], [2, 5]]
    assert sht.thread_partition([3, 4], 2) == [[3, 4], []]
    assert sht.thread_partition([0, 1, 2], 2) == [[0, 2], [1]]
    assert sht.thread_partition([5, 1, 9], 1) == [[1, 5, 9]]
    lay = sht.WorkerLayout.create(gl, 7, 2)
    assert lay.m_sets == sht.assign_m(7, 2) and lay.ring_sets == sht.assign_rings(gl, 2)


def _pack_unpack_emulation(grid, lmax, W):
    """Run the packed exchange of every worker in-process: Legendre rows written through
    row_off (send layout), blocks moved as the all-to-all moves them, rings read through
    m_base/m_stride (receive layout).  Must equal the reference transpose."""
    layout = sht.WorkerLayout.create(grid, lmax, W)
    alm = O.random_alm(lmax, lmax, 5)
    full = O.delta_paired(alm, lmax, lmax, grid.cos_theta)  # [ring][m]
    sends = []
    meta = [sht.exchange_layout(layout, w) for w in range(W)]
    for w in range(W):
        row_off, send_c, recv_c, ring_list, m_base, m_stride = meta[w]
        buf = np.zeros(sum(send_c), np.complex128)
        Mi = layout.m_sets[w]
        for r in range(grid.n_rings):
            buf[row_off[r]:row_off[r] + len(Mi)] = full[r, Mi]
        sends.append((buf, send_c))
    for w in range(W):
        _, _, recv_c, ring_list, m_base, m_stride = meta[w]
        recv = np.concatenate([sends[j][0][sum(sends[j][1][:w]):sum(sends[j][1][:w + 1])] for j in range(W)])
        assert recv.size == sum(recv_c)
        for p, r in enumerate(ring_list):
            row = np.array([recv[m_base[m] + p * m_stride[m]] for m in range(lmax + 1)])
            assert np.array_equal(row, full[r]), (w, r)
    panels = [full[:, layout.m_sets[w]] for w in range(W)]
    ring_panels, vol = O.exchange_m_to_rings(panels, layout.m_sets, layout.ring_sets, lmax)
    for w in range(W):
        assert np.array_equal(ring_panels[w], full[layout.ring_sets[w]])
    assert vol.sum() == 16 * grid.n_rings * (lmax + 1)


@pytest.mark.parametrize("W", [1, 2, 3, 4])
def test_packed_exchange_layout_is_the_reference_transpose(W):
    _pack_unpack_emulation(sht.build_healpix_grid(4), 12, W)
    _pack_unpack_emulation(sht.build_gauss_legendre_grid(8, 16), 7, min(W, 4))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nside, lmax, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = sht.build_healpix_grid(nside)
    layout = sht.WorkerLayout.create(grid, lmax, world)
    row_off, send_c, recv_c, ring_list, m_base, m_stride = sht.exchange_layout(layout, rank)
    alm = O.random_alm(lmax, lmax, 11)
    full = O.delta_paired(alm, lmax, lmax, grid.cos_theta)
    Mi = layout.m_sets[rank]
    send = np.zeros(sum(send_c), np.complex128)
    for r in range(grid.n_rings):
        send[row_off[r]:row_off[r] + len(Mi)] = full[r, Mi]  # only my orders are used
    recv = torch.zeros(2 * sum(recv_c), dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64)),
                           [2 * c for c in recv_c], [2 * c for c in send_c])
    rv = recv.numpy().view(np.complex128)
    out = {}
    for p, r in enumerate(ring_list):
        row = np.array([rv[m_base[m] + p * m_stride[m]] for m in range(lmax + 1)])
        out[int(r)] = O.ring_synthesis(row, int(grid.n_phi[r]), float(grid.phi_0[r]))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_synthesis_over_gloo_world_size_2():
    """distributed_synthesis with 2 workers (distribution.cpp:300-380) through the packed
    all-to-all the GPU path uses, over gloo; bitwise equal to the single-worker result."""
    import torch.multiprocessing as mp
    nside, lmax, W = 4, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, nside, lmax, q)) for r in range(W)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(W):
        _, part = q.get(timeout=120)
        got.update(part)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grid = sht.build_healpix_grid(nside)
    want = O.synthesis(O.random_alm(lmax, lmax, 11), lmax, lmax, grid)
    mp_ = np.concatenate([got[r] for r in range(grid.n_rings)])
    assert np.array_equal(mp_, want)


@pytest.mark.parametrize("policy", ["balanced", "interleaved"])
@pytest.mark.parametrize("nside,W", [(2, 2), (16, 3), (64, 8), (2048, 8)])
def test_multi_gpu_ring_sets_cover_each_ring_once_mirror_closed(policy, nside, W):
    g = sht.build_healpix_grid(nside)
    fn = {"balanced": sht.assign_rings_balanced, "interleaved": sht.assign_rings_interleaved}[policy]
    sets = fn(g, W)
    assert len(sets) == W and all(sets)
    assert sorted(sum(sets, [])) == list(range(g.n_rings))
    for s in sets:  # mirror pairs stay together (the Legendre streams are mirror pairs)
        assert set(s) == {g.n_rings - 1 - r for r in s}
    if policy == "balanced":  # contiguous blocks of north rows, polar blocks shorter
        norths = [sorted(r for r in s if r <= (g.n_rings - 1) // 2) for s in sets]
        assert all(b == list(range(b[0], b[-1] + 1)) for b in norths)
        if nside >= 64:
            assert len(norths[0]) < len(norths[-1])
