"""Host logic of the fused exchange (exchange_m_to_rings / exchange_rings_to_m as direct peer
stores, distribution.cpp:233-298): the store targets `peer_exchange_pointers` hands the kernels
must put every Delta entry exactly where the packed all-to-all would have delivered it.

Device memory is emulated: each worker's send / receive buffer is a numpy array at a fake base
address, and the kernels' stores are replayed with the same address arithmetic
(legendre.cu leg_out: row_ptr[r] + mi row_stride[r]; ringfft.cu delta_out_at: col_ptr[m] +
pos m_stride[m]).  Both synthesis layouts are covered: order-major blocks (the default: a
warp's stores are contiguous runs) and the ring-major blocks shared with map2alm.
The gloo case runs the pointer setup with the base addresses gathered across 2 processes.
"""
import os
import socket

import numpy as np
import pytest

from paper_1106_0159_b200 import sht

BASE = 1 << 40


def code(r, m):
    return complex(1000 * r + m + 1, -(r + 1))


def _fake_bases(layout):
    W = layout.n_workers
    sizes = [sht.exchange_sizes(layout, j) for j in range(W)]
    send = [BASE * (2 * j + 1) for j in range(W)]
    recv = [BASE * (2 * j + 2) for j in range(W)]
    mem = {}
    for j in range(W):
        mem[send[j]] = np.zeros(sizes[j][0], np.complex128)
        mem[recv[j]] = np.zeros(sizes[j][1], np.complex128)
    return send, recv, mem


def _store(mem, addr, val):
    for base, buf in mem.items():
        if base <= addr < base + 16 * buf.size:
            off = addr - base
            assert off % 16 == 0
            buf[off // 16] = val
            return
    raise AssertionError(f"store outside every exchange buffer: {addr:#x}")


def _synthesis_layout(layout, j, order_major):
    """(row_stride, m_base, m_stride) of worker j's alm2map direction"""
    if order_major:
        _, row_stride, m_base, m_stride = sht.exchange_layout_synthesis(layout, j)
        return row_stride, m_base, m_stride
    _, _, _, _, m_base, m_stride = sht.exchange_layout(layout, j)
    return np.ones(layout.n_rings, np.int64), m_base, m_stride


def _replay(layout, send, recv, mem, order_major=True):
    W = layout.n_workers
    ptrs = [sht.peer_exchange_pointers(layout, i, recv, send, order_major) for i in range(W)]
    # alm2map: worker i's Legendre stage stores Delta(r, M_i[mi]) through row_ptr
    for i in range(W):
        row_ptr, _ = ptrs[i]
        row_stride, _, _ = _synthesis_layout(layout, i, order_major)
        for r in range(layout.n_rings):
            for mi, m in enumerate(layout.m_sets[i]):
                _store(mem, int(row_ptr[r]) + 16 * mi * int(row_stride[r]), code(r, m))
    # the ring stage of worker j reads Delta(pos, m) at m_base[m] + pos m_stride[m]
    for j in range(W):
        ring_list = sht.exchange_layout(layout, j)[3]
        _, m_base, m_stride = _synthesis_layout(layout, j, order_major)
        rv = mem[recv[j]]
        for pos, r in enumerate(ring_list):
            for m in range(layout.mmax + 1):
                assert rv[m_base[m] + pos * m_stride[m]] == code(int(r), m), (j, r, m)
    # map2alm: worker j's ring analysis stores Delta^S(pos, m) through col_ptr
    for j in range(W):
        _, col_ptr = ptrs[j]
        _, _, _, ring_list, _, m_stride = sht.exchange_layout(layout, j)
        for pos, r in enumerate(ring_list):
            for m in range(layout.mmax + 1):
                _store(mem, int(col_ptr[m]) + 16 * pos * int(m_stride[m]), code(int(r), m))
    # worker i's Legendre map2alm reads ring r's row of its orders at row_off[r]
    for i in range(W):
        row_off, *_ = sht.exchange_layout(layout, i)
        sv = mem[send[i]]
        for r in range(layout.n_rings):
            for mi, m in enumerate(layout.m_sets[i]):
                assert sv[row_off[r] + mi] == code(r, m), (i, r, m)


@pytest.mark.parametrize("nside,lmax,W,rings", [(2, 5, 1, "blocks"), (4, 12, 2, "blocks"), (4, 12, 3, "blocks"),
                                                 (8, 16, 4, "blocks"), (4, 9, 5, "blocks"), (8, 16, 4, "balanced"),
                                                 (4, 12, 3, "interleaved")])
@pytest.mark.parametrize("order_major", [True, False])
def test_peer_pointers_deliver_like_the_all_to_all(nside, lmax, W, rings, order_major):
    layout = sht.WorkerLayout.create(sht.build_healpix_grid(nside), lmax, W, rings=rings)
    send, recv, mem = _fake_bases(layout)
    _replay(layout, send, recv, mem, order_major)
    for buf in mem.values():  # every slot of every exchange buffer written exactly as planned
        assert np.all(buf != 0)


@pytest.mark.parametrize("W,rings", [(2, "blocks"), (4, "balanced"), (3, "interleaved")])
def test_fused_stores_are_contiguous_runs(W, rings):
    """The NVLink side of both directions coalesces: alm2map's Legendre stores (one order,
    consecutive rings of one owner per warp) land 16 bytes apart in the order-major blocks;
    map2alm's unfold, visiting orders grouped by owner (ascending m_base = the kernels'
    m_order), stores each owner's orders of one ring 16 bytes apart."""
    layout = sht.WorkerLayout.create(sht.build_healpix_grid(16), 40, W, rings=rings)
    send, recv, _ = _fake_bases(layout)
    for i in range(W):
        row_ptr, col_ptr = sht.peer_exchange_pointers(layout, i, recv, send)
        row_stride = sht.exchange_layout_synthesis(layout, i)[1]
        for j in range(W):
            Rj = layout.ring_sets[j]
            for mi in range(len(layout.m_sets[i])):
                addr = [int(row_ptr[r]) + 16 * mi * int(row_stride[r]) for r in Rj]
                assert np.all(np.diff(addr) == 16)
        m_base, m_stride = sht.exchange_layout(layout, i)[4:6]
        order = np.argsort(m_base, kind="stable")
        for j in range(W):  # order owners: a contiguous run of `order` each
            mine = [m for m in order if m in set(layout.m_sets[j])]
            for pos in (0, len(layout.ring_sets[i]) - 1):
                addr = [int(col_ptr[m]) + 16 * pos * int(m_stride[m]) for m in mine]
                assert np.all(np.diff(addr) == 16)


def test_peer_pointers_gauss_legendre_grid():
    layout = sht.WorkerLayout.create(sht.build_gauss_legendre_grid(9, 20), 8, 3)
    send, recv, mem = _fake_bases(layout)
    _replay(layout, send, recv, mem)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layout = sht.WorkerLayout.create(sht.build_healpix_grid(4), 12, world)
    s, r = sht.exchange_sizes(layout, rank)
    mine = (BASE * (2 * rank + 1), BASE * (2 * rank + 2), s, r)
    allb = [None] * world
    dist.all_gather_object(allb, mine)
    row_ptr, col_ptr = sht.peer_exchange_pointers(layout, rank, [b[1] for b in allb], [b[0] for b in allb])
    q.put((rank, row_ptr, col_ptr, allb))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_pointer_setup_over_gloo_world_size_2():
    import torch.multiprocessing as mp
    W = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(W):
        rank, rp, cp, allb = q.get(timeout=120)
        got[rank] = (rp, cp, allb)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    layout = sht.WorkerLayout.create(sht.build_healpix_grid(4), 12, W)
    send, recv, mem = _fake_bases(layout)
    for rank in range(W):
        rp, cp, allb = got[rank]
        assert [b[0] for b in allb] == send and [b[1] for b in allb] == recv
        want_rp, want_cp = sht.peer_exchange_pointers(layout, rank, recv, send)
        assert np.array_equal(rp, want_rp) and np.array_equal(cp, want_cp)
    _replay(layout, send, recv, mem)
