"""GPU: the fused exchange path (Legendre / ring-analysis kernels storing Delta straight into the
consumers' buffers, then the device-side peer barrier) for W workers, bitwise equal to the
single-worker transform (distribution.cpp's worker invariance, test_distribution.cpp:256-311).

Only one GPU is available, so the workers share device 0: in one process (plain addresses,
one context and stream per worker, their barrier kernels waiting on each other across
streams) and in two processes mapping each other's buffers through CUDA IPC with gloo as the
handle transport -- the same calls a multi-GPU run makes over NVLink.
"""
import os
import socket

import numpy as np
import pytest
import torch

from paper_1106_0159_b200 import sht

pytestmark = pytest.mark.gpu


def _single(nside, lmax, seed):
    grid = sht.build_healpix_grid(nside)
    alm_h = sht.random_alm(lmax, lmax, seed)
    c = sht.Context(0)
    c.set_grid(grid)
    c.set_band(lmax, lmax)
    want_map = c.alm2map(alm_h)
    want_alm = c.map2alm(want_map)
    c.close()
    return grid, alm_h, want_map, want_alm


# Workers of one process share the device's hardware work queues: past
# CUDA_DEVICE_MAX_CONNECTIONS (8 by default) a worker's stage kernel can be queued behind
# another worker's waiting barrier kernel, so the one-process case runs in a fresh process with
# 32 connections.  One process per GPU (the multi-GPU layout, and the IPC test below) does not
# share queues between workers.
def _one_process(nside, lmax, W, q, order_major=True):
    try:
        dev = torch.device("cuda", 0)
        grid, alm_h, want_map, want_alm = _single(nside, lmax, 99)
        layout = sht.WorkerLayout.create(grid, lmax, W)
        peers = [None] * W
        xs = []
        for w in range(W):
            c = sht.Context(0)
            c.set_grid(grid)
            c.set_band(lmax, lmax, layout.m_sets[w])
            xs.append(sht.PeerExchange(c, layout, w, peers=peers, order_major=order_major))
        for x in xs:
            x.connect()
        alm = torch.from_numpy(alm_h.view(np.float64)).to(dev)
        mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
        ok = []
        for _ in range(2):  # twice: barrier epochs advance, buffers are rewritten in place
            for x in xs:
                x.alm2map(alm.data_ptr(), mp.data_ptr())
            torch.cuda.synchronize()
            ok.append(bool(np.array_equal(mp.cpu().numpy(), want_map)))
        want_map_d = torch.from_numpy(want_map).to(dev)
        out = torch.zeros(2 * sht.alm_count(lmax, lmax), dtype=torch.float64, device=dev)
        for _ in range(2):
            for x in xs:
                x.map2alm(want_map_d.data_ptr(), out.data_ptr())
            torch.cuda.synchronize()
            ok.append(bool(np.array_equal(out.cpu().numpy().view(np.complex128), want_alm)))
        for x in xs:
            x.close()
        q.put(("ok", ok))
    except Exception as e:  # surfaced in the parent
        q.put(("error", repr(e)))


@pytest.mark.parametrize("nside,lmax,W,order_major", [(8, 16, 2, True), (32, 64, 3, True), (64, 128, 4, True),
                                                      (128, 256, 4, True), (128, 256, 8, True),
                                                      (64, 128, 4, False)])
def test_fused_exchange_one_process(nside, lmax, W, order_major):
    import torch.multiprocessing as mp
    os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"  # inherited by the spawned process
    os.environ["SHTC_FFT_AUX"] = "2"  # W contexts x 3 ring-stage streams stay within 32 queues
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_one_process, args=(nside, lmax, W, q, order_major))
        p.start()
        status, res = q.get(timeout=300)
        p.join(timeout=60)
    finally:
        os.environ.pop("CUDA_DEVICE_MAX_CONNECTIONS", None)
        os.environ.pop("SHTC_FFT_AUX", None)
    assert status == "ok", res
    assert all(res), res
    assert p.exitcode == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, nside, lmax, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    try:
        dev = torch.device("cuda", 0)
        grid = sht.build_healpix_grid(nside)
        layout = sht.WorkerLayout.create(grid, lmax, world)
        c = sht.Context(0)
        c.set_grid(grid)
        c.set_band(lmax, lmax, layout.m_sets[rank])
        x = sht.PeerExchange(c, layout, rank, all_gather=all_gather)
        alm = torch.from_numpy(sht.random_alm(lmax, lmax, 5).view(np.float64)).to(dev)
        mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
        x.alm2map(alm.data_ptr(), mp.data_ptr())
        torch.cuda.synchronize()
        dist.barrier()
        # this worker's rings of the map (the others stay zero)
        ring_map = mp.cpu().numpy().copy()
        out = torch.zeros(2 * sht.alm_count(lmax, lmax), dtype=torch.float64, device=dev)
        full = torch.from_numpy(q_full_map(grid, lmax)).to(dev)
        x.map2alm(full.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, ring_map, out.cpu().numpy().view(np.complex128).copy()))
        x.close()
        c.close()
    finally:
        dist.barrier()
        dist.destroy_process_group()


def q_full_map(grid, lmax):
    return sht.gaussian_map(grid.n_pix, 2026)


def test_fused_exchange_two_processes_ipc():
    import torch.multiprocessing as mp
    nside, lmax, W = 32, 64, 2
    grid, alm_h, _, _ = _single(nside, lmax, 5)
    c = sht.Context(0)
    c.set_grid(grid)
    c.set_band(lmax, lmax)
    want_map = c.alm2map(sht.random_alm(lmax, lmax, 5))
    want_alm = c.map2alm(q_full_map(grid, lmax))
    c.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, W, port, nside, lmax, q)) for r in range(W)]
    for p in procs:
        p.start()
    parts = {}
    for _ in range(W):
        rank, ring_map, a = q.get(timeout=300)
        parts[rank] = (ring_map, a)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    layout = sht.WorkerLayout.create(grid, lmax, W)
    mp_ = np.zeros(grid.n_pix)
    alm = np.zeros(sht.alm_count(lmax, lmax), np.complex128)
    for w in range(W):
        ring_map, a = parts[w]
        mp_ += ring_map  # disjoint ring sets
        for m in layout.m_sets[w]:
            o = sht.alm_offset(m, lmax)
            alm[o:o + lmax - m + 1] = a[o:o + lmax - m + 1]
    assert np.array_equal(mp_, want_map)
    assert np.array_equal(alm, want_alm)
