"""Python host mirror of the reference's SHT operator interface, backed by libshtc (CUDA).

Names, argument meaning and error classes follow /root/reference/proj/include/sht:
  build_healpix_grid / build_gauss_legendre_grid / gauss_legendre_nodes   grid.hpp:45-58
  symmetric_ring_pairs                                                     grid.hpp:62-63
  AlmSet count / offset (m-major triangle)                                 alm.hpp:16-35
  synthesis / analysis (alm2map / map2alm)                                 transforms.hpp:73-79
  compute_delta_a / compute_delta_a_ring_major / accumulate_alm /
  accumulate_alm_partial / reduce_partials                                 transforms.hpp:32-69
  splitmix64_at / uniform_pm1 / random_alm                                 experiment.hpp:14-25
  assign_m / assign_rings / thread_partition / WorkerLayout                distribution.hpp:15-40
Every transform runs on the GPU through the C ABI; the geometry, layouts and input
generators are host-side bookkeeping (they are not on the hot path).
std::invalid_argument maps to ValueError, std::domain_error to ArithmeticError.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import GroupTiming, Timing, check, lib

# ----------------------------------------------------------------------------------------
# containers and geometry
# ----------------------------------------------------------------------------------------


def alm_count(lmax: int, mmax: int) -> int:
    """AlmSet::count (alm.cpp:13-16)."""
    return (mmax + 1) * (lmax + 1) - mmax * (mmax + 1) // 2


def alm_offset(m: int, lmax: int) -> int:
    """AlmSet::offset (alm.hpp:27-30)."""
    return m * (lmax + 1) - m * (m - 1) // 2


def alm_index(l: int, m: int, lmax: int) -> int:
    return alm_offset(m, lmax) + (l - m)


@dataclass
class PixelGrid:
    """sht::PixelGrid (grid.hpp:27-37) as plain ring arrays."""

    scheme: str
    nside: int
    cos_theta: np.ndarray
    n_phi: np.ndarray
    phi_0: np.ndarray
    weight: np.ndarray
    pixel_offset: np.ndarray = field(default=None)

    def __post_init__(self):
        self.cos_theta = np.ascontiguousarray(self.cos_theta, dtype=np.float64)
        self.n_phi = np.ascontiguousarray(self.n_phi, dtype=np.int32)
        self.phi_0 = np.ascontiguousarray(self.phi_0, dtype=np.float64)
        self.weight = np.ascontiguousarray(self.weight, dtype=np.float64)
        if self.pixel_offset is None:
            self.pixel_offset = np.concatenate(
                [[0], np.cumsum(self.n_phi.astype(np.int64))[:-1]]).astype(np.int64)
        self.pixel_offset = np.ascontiguousarray(self.pixel_offset, dtype=np.int64)

    @property
    def n_rings(self) -> int:
        return int(self.cos_theta.shape[0])

    @property
    def n_pix(self) -> int:
        return int(self.n_phi.astype(np.int64).sum())

    def cos_thetas(self) -> np.ndarray:
        return self.cos_theta.copy()


def build_healpix_grid(nside: int) -> PixelGrid:
    """HEALPix ring scheme (grid.cpp:23-67)."""
    if nside < 1:
        raise ValueError("healpix grid: nside must be >= 1")
    n_rings = 4 * nside - 1
    npix = 12 * nside * nside
    z = np.zeros(n_rings)
    nphi = np.zeros(n_rings, np.int32)
    p0 = np.zeros(n_rings)
    w = np.full(n_rings, 4.0 * math.pi / float(npix))
    for i in range(1, 2 * nside + 1):
        if i < nside:
            nphi[i - 1] = 4 * i
            z[i - 1] = 1.0 - float(i) * i / (3.0 * nside * nside)
            p0[i - 1] = math.pi / (4.0 * i)
        else:
            nphi[i - 1] = 4 * nside
            z[i - 1] = 4.0 / 3.0 - 2.0 * i / (3.0 * nside)
            p0[i - 1] = math.pi / (4.0 * nside) if (i - nside) % 2 == 0 else 0.0
    for i in range(2 * nside + 1, n_rings + 1):
        src = (4 * nside - i) - 1
        nphi[i - 1] = nphi[src]
        p0[i - 1] = p0[src]
        z[i - 1] = -z[src]
    return PixelGrid("healpix-ring", nside, z, nphi, p0, w)


def gauss_legendre_nodes(n: int):
    """Nodes (descending) and weights by Newton iteration on P_n (grid.cpp:69-104)."""
    if n < 1:
        raise ValueError("gauss_legendre_nodes: n must be >= 1")
    x = np.zeros(n)
    w = np.zeros(n)
    for i in range((n + 1) // 2):
        t = math.cos(math.pi * (i + 0.75) / (n + 0.5))
        dp = 0.0
        for _ in range(100):
            p0, p1 = 1.0, t
            for l in range(2, n + 1):
                p0, p1 = p1, ((2.0 * l - 1.0) * t * p1 - (l - 1.0) * p0) / l
            dp = n * (p0 - t * p1) / (1.0 - t * t)
            dt = p1 / dp
            t -= dt
            if abs(dt) < 1e-15:
                break
        else:
            raise RuntimeError("gauss_legendre_nodes: Newton iteration failed")
        x[i] = t
        w[i] = 2.0 / ((1.0 - t * t) * dp * dp)
        x[n - 1 - i] = -t
        w[n - 1 - i] = w[i]
    if n % 2 == 1:
        x[n // 2] = 0.0
    return x, w


def build_gauss_legendre_grid(n_rings: int, n_phi: int) -> PixelGrid:
    """Gauss-Legendre grid (grid.cpp:106-131)."""
    if n_rings < 1:
        raise ValueError("gauss-legendre grid: n_rings must be >= 1")
    if n_phi < 1:
        raise ValueError("gauss-legendre grid: n_phi must be >= 1")
    x, glw = gauss_legendre_nodes(n_rings)
    return PixelGrid("gauss-legendre", 0, x, np.full(n_rings, n_phi, np.int32),
                     np.zeros(n_rings), 2.0 * math.pi / n_phi * glw)


def symmetric_ring_pairs(grid: PixelGrid):
    """grid.cpp:133-151."""
    n = grid.n_rings
    pairs = []
    for k in range(n // 2):
        j = n - 1 - k
        if grid.n_phi[k] != grid.n_phi[j] or abs(grid.cos_theta[k] + grid.cos_theta[j]) > 1e-14:
            raise ValueError("symmetric_ring_pairs: grid is not mirror symmetric")
        pairs.append((k, j))
    if n % 2 == 1:
        if abs(grid.cos_theta[n // 2]) > 1e-14:
            raise ValueError("symmetric_ring_pairs: central ring is off the equator")
        pairs.append((n // 2, None))
    return pairs


# ----------------------------------------------------------------------------------------
# synthetic inputs (experiment.cpp:11-33)
# ----------------------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64_at(seed, index):
    """Counter-based splitmix64 (experiment.cpp:11-16), vectorised over index."""
    with np.errstate(over="ignore"):
        idx = np.asarray(index, dtype=np.uint64)
        z = np.uint64(seed) + (idx + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed, index):
    u = ((splitmix64_at(seed, index) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    return 2.0 * u - 1.0


def random_alm(lmax: int, mmax: int, seed: int) -> np.ndarray:
    """Re, Im i.i.d. uniform(-1,1), Im a_l0 = 0 (experiment.cpp:24-33)."""
    n = alm_count(lmax, mmax)
    k = np.arange(n, dtype=np.uint64)
    a = uniform_pm1(seed, 2 * k) + 1j * uniform_pm1(seed, 2 * k + np.uint64(1))
    a[: lmax + 1] = a[: lmax + 1].real  # m == 0 block
    return a


def gaussian_alm(lmax: int, mmax: int, seed: int) -> np.ndarray:
    """N(0,1) re/im by Box-Muller on the same counter stream, Im a_l0 = 0."""
    n = alm_count(lmax, mmax)
    k = np.arange(n, dtype=np.uint64)
    u1 = ((splitmix64_at(seed, 2 * k) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = ((splitmix64_at(seed, 2 * k + np.uint64(1)) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    a = r * np.cos(2 * np.pi * u2) + 1j * r * np.sin(2 * np.pi * u2)
    a[: lmax + 1] = a[: lmax + 1].real
    return a


def gaussian_map(n_pix: int, seed: int) -> np.ndarray:
    k = np.arange(n_pix, dtype=np.uint64)
    u1 = ((splitmix64_at(seed, 2 * k) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = ((splitmix64_at(seed, 2 * k + np.uint64(1)) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * u2)


# ----------------------------------------------------------------------------------------
# distribution layouts (distribution.cpp:82-171) — host bookkeeping for multi-GPU runs
# ----------------------------------------------------------------------------------------
def assign_m(mmax: int, n_workers: int):
    if mmax < 0:
        raise ValueError("assign_m: mmax must be >= 0")
    if n_workers < 1:
        raise ValueError("assign_m: n_workers must be >= 1")
    if n_workers > 1 and n_workers > (mmax + 1) // 2:
        raise ValueError("assign_m: n_workers > mmax/2")
    sets = [[] for _ in range(n_workers)]
    lo, hi, w = 0, mmax, 0
    while lo < hi:
        sets[w] += [lo, hi]
        lo += 1
        hi -= 1
        w = (w + 1) % n_workers
    if lo == hi:
        sets[w].append(lo)
    return [sorted(s) for s in sets]


def assign_rings(grid: PixelGrid, n_workers: int):
    r_n = grid.n_rings
    if n_workers < 1:
        raise ValueError("assign_rings: n_workers must be >= 1")
    if r_n < 1:
        raise ValueError("assign_rings: empty grid")
    if n_workers == 1:
        return [list(range(r_n))]
    if 2 * n_workers > r_n:
        raise ValueError("assign_rings: n_workers > n_rings/2")
    h = (r_n + 1) // 2
    q, rem = divmod(h, n_workers)
    sets, row = [], 0
    for w in range(n_workers):
        s = []
        for _ in range(q + (1 if w < rem else 0)):
            s.append(row)
            if r_n - 1 - row != row:
                s.append(r_n - 1 - row)
            row += 1
        sets.append(sorted(s))
    return sets


def assign_rings_interleaved(grid: PixelGrid, n_workers: int):
    """Ring sets of the multi-GPU runs: mirror pairs (north k, south R-1-k) dealt round-robin,
    so every worker gets the same mix of polar-cap and belt rings.  The reference's
    contiguous blocks (assign_rings) give the polar workers all the small, aliasing cap rings,
    whose ring stage costs several times the belt rings' per pixel (measured at C4, 8 workers:
    0.56 against 0.17 ms).  Results are partition-invariant, as in the reference."""
    r_n = grid.n_rings
    if n_workers < 1:
        raise ValueError("assign_rings: n_workers must be >= 1")
    if r_n < 1:
        raise ValueError("assign_rings: empty grid")
    if n_workers == 1:
        return [list(range(r_n))]
    if 2 * n_workers > r_n:
        raise ValueError("assign_rings: n_workers > n_rings/2")
    h = (r_n + 1) // 2
    sets = [[] for _ in range(n_workers)]
    for row in range(h):
        s = sets[row % n_workers]
        s.append(row)
        if r_n - 1 - row != row:
            s.append(r_n - 1 - row)
    return [sorted(s) for s in sets]


CAP_WEIGHT = float(os.environ.get("SHT_CAP_WEIGHT", "3.0"))


def assign_rings_balanced(grid: PixelGrid, n_workers: int):
    """Ring sets of the multi-GPU runs: contiguous blocks of mirror pairs, as assign_rings, but
    of equal ring-stage cost instead of equal ring count.  A ring shorter than the longest
    (HEALPix polar caps: aliasing folds over many wraps, Bluestein sizes, small latency-bound
    classes) weighs CAP_WEIGHT = 3 belt rings -- measured at C4 with 8 workers: 0.34-0.59 us
    per cap ring, 0.14-0.24 us per belt ring.
    Results are partition-invariant, as in the reference."""
    r_n = grid.n_rings
    if n_workers < 1:
        raise ValueError("assign_rings: n_workers must be >= 1")
    if r_n < 1:
        raise ValueError("assign_rings: empty grid")
    if n_workers == 1:
        return [list(range(r_n))]
    if 2 * n_workers > r_n:
        raise ValueError("assign_rings: n_workers > n_rings/2")
    h = (r_n + 1) // 2
    nphi = np.asarray(grid.n_phi)
    top = int(nphi.max())
    w = np.where(nphi[:h] < top, CAP_WEIGHT, 1.0)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    sets, row = [], 0
    for k in range(n_workers):
        # rows [row, end): cumulative weight up to the k+1-th share, at least one row, and
        # leave one row for each later worker
        end = int(np.searchsorted(cum, total * (k + 1) / n_workers, side="left"))
        end = max(row + 1, min(end, h - (n_workers - 1 - k)))
        if k == n_workers - 1:
            end = h
        s = []
        for r in range(row, end):
            s.append(r)
            if r_n - 1 - r != r:
                s.append(r_n - 1 - r)
        sets.append(sorted(s))
        row = end
    return sets


def thread_partition(m_set, n_threads: int):
    if n_threads <= 0:
        raise ValueError("thread_partition: n_threads must be >= 1")
    ms = sorted(m_set)
    sets = [[] for _ in range(n_threads)]
    if not ms:
        return sets
    top = ms[-1]
    load = [0] * n_threads
    lo, hi, t = 0, len(ms) - 1, 0
    while lo < hi:
        sets[t] += [ms[lo], ms[hi]]
        load[t] += (top + 1 - ms[lo]) + (top + 1 - ms[hi])
        lo += 1
        hi -= 1
        t = (t + 1) % n_threads
    if lo == hi:
        best = min(range(n_threads), key=lambda j: (load[j], j))
        sets[best].append(ms[lo])
    return [sorted(s) for s in sets]


@dataclass
class WorkerLayout:
    n_workers: int
    mmax: int
    n_rings: int
    m_sets: list
    ring_sets: list

    @staticmethod
    def create(grid: PixelGrid, mmax: int, n_workers: int, rings: str = "blocks") -> "WorkerLayout":
        """rings="blocks": the reference's assign_rings; "balanced": assign_rings_balanced (the
        multi-GPU bench's choice); "interleaved": assign_rings_interleaved."""
        m_sets = [list(range(mmax + 1))] if n_workers == 1 else assign_m(mmax, n_workers)
        ring_sets = {"blocks": assign_rings, "interleaved": assign_rings_interleaved,
                     "balanced": assign_rings_balanced}[rings](grid, n_workers)
        return WorkerLayout(n_workers, mmax, grid.n_rings, m_sets, ring_sets)


def exchange_layout(layout: WorkerLayout, rank: int):
    """Packed all-to-all layouts of one worker (exchange_m_to_rings, distribution.cpp:233-298).

    Send side (Legendre output, alm2map): rows grouped by destination worker j, each block
    [|R_j| rows x |M_rank| cols] contiguous; row_off[r] = complex offset of ring r's row.
    Receive side (fold input): block from source j is [|R_rank| x |M_j|]; order m of M_j lives
    at m_base[m] + pos * m_stride[m] for ring position pos in R_rank.
    Returns (row_off, send_counts, recv_counts, ring_list, m_base, m_stride) in complex units.
    The same layouts serve map2alm in reverse (analysis writes the recv-shaped blocks per
    destination owner, the Legendre stage reads rows through row_off).
    """
    W = layout.n_workers
    Mi = layout.m_sets[rank]
    row_off = np.zeros(layout.n_rings, np.int64)
    send_counts = []
    off = 0
    for j in range(W):
        Rj = layout.ring_sets[j]
        for p, r in enumerate(Rj):
            row_off[r] = off + p * len(Mi)
        send_counts.append(len(Rj) * len(Mi))
        off += len(Rj) * len(Mi)
    Ri = layout.ring_sets[rank]
    m_base = np.zeros(layout.mmax + 1, np.int64)
    m_stride = np.zeros(layout.mmax + 1, np.int64)
    recv_counts = []
    off = 0
    for j in range(W):
        Mj = layout.m_sets[j]
        for c, m in enumerate(Mj):
            m_base[m] = off + c
            m_stride[m] = len(Mj)
        recv_counts.append(len(Ri) * len(Mj))
        off += len(Ri) * len(Mj)
    return row_off, send_counts, recv_counts, np.asarray(Ri, np.int32), m_base, m_stride


def exchange_layout_synthesis(layout: WorkerLayout, rank: int):
    """Order-major synthesis layout of one worker (shtc_set_exchange_layout_synthesis): the
    same blocks and offsets as exchange_layout, each block [orders x rings].

    Send side (Legendre output): ring r = R_j[p] of this worker's order index c at
    row_off[r] + c * row_stride[r] with row_off[r] = block offset + p, row_stride[r] = |R_j|,
    so a warp's stores (one order, consecutive rings) are contiguous.  Receive side: order m
    (index c in M_j) of ring position p at m_base[m] + p, m_base[m] = block offset + c |R_rank|,
    m_stride = 1.  Returns (row_off, row_stride, m_base, m_stride) in complex units."""
    W = layout.n_workers
    Mi = layout.m_sets[rank]
    row_off = np.zeros(layout.n_rings, np.int64)
    row_stride = np.ones(layout.n_rings, np.int64)
    off = 0
    for j in range(W):
        Rj = layout.ring_sets[j]
        for p, r in enumerate(Rj):
            row_off[r] = off + p
            row_stride[r] = len(Rj)
        off += len(Rj) * len(Mi)
    Ri = layout.ring_sets[rank]
    m_base = np.zeros(layout.mmax + 1, np.int64)
    m_stride = np.ones(layout.mmax + 1, np.int64)
    off = 0
    for j in range(W):
        Mj = layout.m_sets[j]
        for c, m in enumerate(Mj):
            m_base[m] = off + c * len(Ri)
        off += len(Ri) * len(Mj)
    return row_off, row_stride, m_base, m_stride


def exchange_sizes(layout: WorkerLayout, rank: int):
    """(send, recv) buffer sizes of one worker in complex elements."""
    Mi, Ri = len(layout.m_sets[rank]), len(layout.ring_sets[rank])
    send = sum(len(Rj) for Rj in layout.ring_sets) * Mi
    recv = Ri * sum(len(Mj) for Mj in layout.m_sets)
    return send, recv


def peer_exchange_pointers(layout: WorkerLayout, rank: int, recv_bases, send_bases,
                           order_major: bool = True):
    """Store targets of worker `rank` on the fused exchange path (shtc_set_exchange_peers).

    recv_bases[j] / send_bases[j]: device addresses (valid in this process) of worker j's
    receive / send buffers, laid out as exchange_layout (map2alm) and, with order_major,
    exchange_layout_synthesis (alm2map) describe.  Returns
      row_ptr[r]: where ring r's element of this worker's first order goes in the ring owner's
                  receive buffer (the block from source `rank`: position pos, further orders
                  |R_owner| apart; ring-major without order_major: row pos * |M_rank|);
      col_ptr[m]: order m's column for this worker's ring position 0 in the order owner's send
                  buffer (the block for destination `rank`), rows |M_owner| apart (m_stride).
    Byte addresses as uint64 (16-byte complex elements)."""
    W = layout.n_workers
    Msz = [len(M) for M in layout.m_sets]
    Rsz = [len(R) for R in layout.ring_sets]
    row_ptr = np.zeros(layout.n_rings, np.uint64)
    for j in range(W):
        off = sum(Rsz[j] * Msz[s] for s in range(rank))  # block of source `rank` in j's recv
        for pos, r in enumerate(layout.ring_sets[j]):
            row_ptr[r] = int(recv_bases[j]) + 16 * (off + (pos if order_major else pos * Msz[rank]))
    col_ptr = np.zeros(layout.mmax + 1, np.uint64)
    for i in range(W):
        soff = sum(Rsz[d] * Msz[i] for d in range(rank))  # block for destination `rank` in i's send
        for c, m in enumerate(layout.m_sets[i]):
            col_ptr[m] = int(send_bases[i]) + 16 * (soff + c)
    return row_ptr, col_ptr


# ----------------------------------------------------------------------------------------
# GPU context
# ----------------------------------------------------------------------------------------
def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Context:
    """One GPU's transform state (geometry, band, cached plans) — the C ABI shtc_ctx."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().shtc_create(int(device), C.byref(self._h)))
        self.device = device
        self.grid = None
        self.lmax = self.mmax = None

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().shtc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        check(rc, self._h)

    def set_stream(self, stream_ptr: int | None):
        self._check(lib().shtc_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def set_grid(self, grid: PixelGrid, mirror: bool = True):
        self._check(lib().shtc_set_grid(self._h, grid.n_rings, _p(grid.cos_theta), _p(grid.n_phi),
                                        _p(grid.phi_0), _p(grid.weight), _p(grid.pixel_offset),
                                        int(bool(mirror))))
        self.grid = grid

    def set_band(self, lmax: int, mmax: int, ms=None):
        if ms is None:
            self._check(lib().shtc_set_band(self._h, lmax, mmax, 0, None))
        else:
            ms = np.ascontiguousarray(ms, np.int32)
            self._check(lib().shtc_set_band(self._h, lmax, mmax, len(ms), _p(ms)))
        self.lmax, self.mmax = lmax, mmax

    def set_ladder(self, enabled: bool = True):
        """ScaleLadder::standard() (True) or ScaleLadder::unscaled() (False)."""
        self._check(lib().shtc_set_ladder(self._h, int(bool(enabled))))

    def plan(self) -> float:
        t = C.c_double()
        self._check(lib().shtc_plan(self._h, C.byref(t)))
        return t.value

    def plan_stats(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(lib().shtc_plan_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        d, e, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(lib().shtc_plan_phase_stats(self._h, C.byref(d), C.byref(e), C.byref(f)))
        g, h = C.c_uint64(), C.c_uint64()
        self._check(lib().shtc_plan_executed(self._h, C.byref(g), C.byref(h)))
        return {"nominal": a.value, "executed": b.value, "useful": c.value,
                "prefix": d.value, "checked": e.value, "fast": f.value,
                "executed_alm2map": g.value, "executed_map2alm": h.value}

    # host-buffer transforms ---------------------------------------------------------
    def alm2map(self, alm: np.ndarray, out: np.ndarray | None = None, timing: bool = False):
        alm = np.ascontiguousarray(alm, np.complex128)
        if alm.size != alm_count(self.lmax, self.mmax):
            raise ValueError("alm2map: coefficient count != AlmSet::count(lmax, mmax)")
        mp = out if out is not None else np.empty(self.grid.n_pix)
        t = Timing()
        self._check(lib().shtc_alm2map(self._h, _p(alm), _p(mp), C.byref(t)))
        return (mp, t.as_dict()) if timing else mp

    def map2alm(self, mp: np.ndarray, out: np.ndarray | None = None, timing: bool = False):
        mp = np.ascontiguousarray(mp, np.float64)
        if mp.size != self.grid.n_pix:
            raise ValueError("analysis: pixel count != grid")
        alm = out if out is not None else np.empty(alm_count(self.lmax, self.mmax), np.complex128)
        t = Timing()
        self._check(lib().shtc_map2alm(self._h, _p(mp), _p(alm), C.byref(t)))
        return (alm, t.as_dict()) if timing else alm

    # device-pointer entry points (ints are raw CUDA pointers, e.g. torch.data_ptr()) --
    def alm2map_dev(self, alm_ptr: int, map_ptr: int, timing: bool = False):
        t = Timing()
        self._check(lib().shtc_alm2map_dev(self._h, C.c_void_p(alm_ptr), C.c_void_p(map_ptr),
                                           C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def map2alm_dev(self, map_ptr: int, alm_ptr: int, timing: bool = False):
        t = Timing()
        self._check(lib().shtc_map2alm_dev(self._h, C.c_void_p(map_ptr), C.c_void_p(alm_ptr),
                                           C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def set_exchange_layout(self, row_off=None, ring_list=None, m_base=None, m_stride=None):
        if row_off is None:
            self._check(lib().shtc_set_exchange_layout(self._h, None, 0, None, None, None))
            return
        ro = np.ascontiguousarray(row_off, np.int64)
        rl = np.ascontiguousarray(ring_list, np.int32)
        mb = np.ascontiguousarray(m_base, np.int64)
        mst = np.ascontiguousarray(m_stride, np.int64)
        self._check(lib().shtc_set_exchange_layout(self._h, _p(ro), len(rl), _p(rl), _p(mb), _p(mst)))

    def set_exchange_layout_synthesis(self, row_off=None, row_stride=None, m_base=None, m_stride=None):
        if row_off is None:
            self._check(lib().shtc_set_exchange_layout_synthesis(self._h, None, None, None, None))
            return
        a = [np.ascontiguousarray(x, np.int64) for x in (row_off, row_stride, m_base, m_stride)]
        self._check(lib().shtc_set_exchange_layout_synthesis(self._h, *[_p(x) for x in a]))

    def legendre_alm2map_dev(self, alm_ptr, delta_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_legendre_alm2map_dev(self._h, C.c_void_p(alm_ptr), C.c_void_p(delta_ptr),
                                                    C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def legendre_map2alm_dev(self, delta_ptr, alm_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_legendre_map2alm_dev(self._h, C.c_void_p(delta_ptr), C.c_void_p(alm_ptr),
                                                    C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def ring_synthesis_dev(self, delta_ptr, map_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_ring_synthesis_dev(self._h, C.c_void_p(delta_ptr), C.c_void_p(map_ptr),
                                                  C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def ring_analysis_dev(self, map_ptr, delta_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_ring_analysis_dev(self._h, C.c_void_p(map_ptr), C.c_void_p(delta_ptr),
                                                 C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    # fused exchange over peer memory (see PeerExchange) ---------------------------------
    def set_exchange_peers(self, row_ptr=None, col_ptr=None):
        if row_ptr is None:
            self._check(lib().shtc_set_exchange_peers(self._h, None, None))
            return
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        cp = np.ascontiguousarray(col_ptr, np.uint64)
        self._check(lib().shtc_set_exchange_peers(self._h, _p(rp), _p(cp)))

    def legendre_alm2map_peer(self, alm_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_legendre_alm2map_peer(self._h, C.c_void_p(alm_ptr), C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def ring_analysis_peer(self, map_ptr, timing=False):
        t = Timing()
        self._check(lib().shtc_ring_analysis_peer(self._h, C.c_void_p(map_ptr), C.byref(t) if timing else None))
        return t.as_dict() if timing else None

    def copy_orders(self, src_ptr: int, dst_ptr: int, to_device: bool):
        """This context's orders between two full a_lm triangles (host <-> device, async on
        the context stream)."""
        self._check(lib().shtc_copy_orders(self._h, C.c_void_p(src_ptr), C.c_void_p(dst_ptr),
                                           1 if to_device else 0))

    def peer_barrier(self, rank: int, n_workers: int, flag_ptrs, epoch: int):
        f = np.ascontiguousarray(flag_ptrs, np.uint64)
        self._check(lib().shtc_peer_barrier(self._h, rank, n_workers, _p(f), C.c_uint32(epoch & 0xFFFFFFFF)))

    # Legendre-stage operators ----------------------------------------------------------
    def delta_a(self, alm, lmax, mmax, x, ms):
        alm = np.ascontiguousarray(alm, np.complex128)
        x = np.ascontiguousarray(x, np.float64)
        ms = np.ascontiguousarray(ms, np.int32)
        out = np.zeros((len(x), len(ms)), np.complex128)
        steps = C.c_uint64(0)
        self._check(lib().shtc_delta_a(self._h, _p(alm), lmax, mmax, len(x), _p(x), len(ms), _p(ms),
                                       _p(out), C.byref(steps)))
        return out, steps.value

    def accumulate_alm(self, delta, x, ms, lmax, mmax, alm_inout=None):
        d = np.ascontiguousarray(delta, np.complex128)
        x = np.ascontiguousarray(x, np.float64)
        ms = np.ascontiguousarray(ms, np.int32)
        out = (np.zeros(alm_count(lmax, mmax), np.complex128) if alm_inout is None
               else np.ascontiguousarray(alm_inout, np.complex128).copy())
        steps = C.c_uint64(0)
        self._check(lib().shtc_accumulate_alm(self._h, _p(d), len(x), _p(x), len(ms), _p(ms), lmax, mmax,
                                              _p(out), C.byref(steps)))
        return out, steps.value


_DEFAULT = {}


# ----------------------------------------------------------------------------------------
# fused exchange over peer memory
# ----------------------------------------------------------------------------------------
def dev_alloc(device: int, nbytes: int) -> int:
    p = C.c_void_p()
    check(lib().shtc_dev_alloc(int(device), int(nbytes), C.byref(p)))
    return int(p.value)


def dev_free(ptr: int):
    check(lib().shtc_dev_free(C.c_void_p(ptr)))


def ipc_handle(ptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    check(lib().shtc_ipc_handle(C.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(device: int, handle: bytes) -> int:
    p = C.c_void_p()
    check(lib().shtc_ipc_open(int(device), C.c_char_p(handle), C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int):
    check(lib().shtc_ipc_close(C.c_void_p(ptr)))


class PeerExchange:
    """One worker's side of the fused exchange (distributed_synthesis/analysis, distribution.cpp:
    300-490, with exchange_m_to_rings / rings_to_m as direct peer stores).

    Owns this worker's send buffer (Legendre side: a_lm orders x all rings), receive buffer
    (ring side: its rings x all orders) and barrier flags, all from shtc_dev_alloc; maps the
    other workers' buffers through CUDA IPC (`all_gather(obj) -> list over ranks`, e.g. over
    torch.distributed) or, for workers of one process, takes their addresses directly.

        alm2map: legendre_alm2map_peer(alm) -> barrier -> ring_synthesis_dev(recv, map)
        map2alm: ring_analysis_peer(map) -> barrier -> legendre_map2alm_dev(send, alm)
    """

    def __init__(self, ctx: Context, layout: WorkerLayout, rank: int, all_gather=None, peers=None,
                 order_major: bool = True):
        self.ctx, self.layout, self.rank = ctx, layout, rank
        self.order_major = order_major
        W = layout.n_workers
        self.n = W
        send_c, recv_c = exchange_sizes(layout, rank)
        dev = ctx.device
        self.send = dev_alloc(dev, 16 * max(send_c, 1))
        self.recv = dev_alloc(dev, 16 * max(recv_c, 1))
        self.flags = dev_alloc(dev, 4 * W)
        self.epoch = 0
        self._last = None
        self._opened = []
        mine = (self.send, self.recv, self.flags)
        if peers is not None:                       # workers in one process: plain addresses
            self._peers = peers
            self._peers[rank] = mine
            return
        hs = all_gather((ipc_handle(self.send), ipc_handle(self.recv), ipc_handle(self.flags)))
        addrs = []
        for j, h in enumerate(hs):
            if j == rank:
                addrs.append(mine)
                continue
            a = tuple(ipc_open(dev, x) for x in h)
            self._opened += list(a)
            addrs.append(a)
        self._peers = addrs
        self.connect()

    def connect(self):
        """Set the layout and the peer store targets on the context (after every worker of
        a single-process group is constructed)."""
        row_off, send_c, recv_c, ring_list, m_base, m_stride = exchange_layout(self.layout, self.rank)
        self.ctx.set_exchange_layout(row_off, ring_list, m_base, m_stride)
        # alm2map blocks order-major: every warp's NVLink stores are contiguous runs
        # (order_major=False keeps the ring-major blocks of map2alm, the comparison layout)
        if self.order_major:
            self.ctx.set_exchange_layout_synthesis(*exchange_layout_synthesis(self.layout, self.rank))
        send_b = [p[0] for p in self._peers]
        recv_b = [p[1] for p in self._peers]
        row_ptr, col_ptr = peer_exchange_pointers(self.layout, self.rank, recv_b, send_b, self.order_major)
        self.ctx.set_exchange_peers(row_ptr, col_ptr)
        self._flag_ptrs = np.array([p[2] for p in self._peers], np.uint64)
        # build every plan now: no allocation or synchronising call may run once a worker's
        # barrier kernel is waiting for the others
        self.ctx.plan()

    def barrier(self):
        self.epoch += 1
        self.ctx.peer_barrier(self.rank, self.n, self._flag_ptrs, self.epoch)

    # Write-after-read: alm2map's peer stores land in the other workers' `recv`, which their
    # previous alm2map's ring synthesis may still be reading (map2alm: `send` and the Legendre
    # stage).  Alternating directions are ordered by the other direction's barrier; a repeated
    # direction passes one extra barrier before its peer stores.
    def alm2map(self, alm_ptr: int, map_ptr: int, timing=False):
        if self._last == "alm2map":
            self.barrier()
        self._last = "alm2map"
        t1 = self.ctx.legendre_alm2map_peer(alm_ptr, timing)
        self.barrier()
        t2 = self.ctx.ring_synthesis_dev(self.recv, map_ptr, timing)
        return (t1, t2) if timing else None

    def map2alm(self, map_ptr: int, alm_ptr: int, timing=False):
        if self._last == "map2alm":
            self.barrier()
        self._last = "map2alm"
        t1 = self.ctx.ring_analysis_peer(map_ptr, timing)
        self.barrier()
        t2 = self.ctx.legendre_map2alm_dev(self.send, alm_ptr, timing)
        return (t2, t1) if timing else None

    def close(self):
        for p in self._opened:
            ipc_close(p)
        self._opened = []
        for p in (self.send, self.recv, self.flags):
            if p:
                dev_free(p)
        self.send = self.recv = self.flags = 0


class Group:
    """Single-process multi-GPU transforms: W workers, worker i on devices[i] (default i mod the
    device count) -- the C ABI shtc_group (distributed_synthesis / distributed_analysis,
    distribution.cpp:300-490).  exchange="peer": the stage kernels store Delta straight into
    the other workers' buffers (NVLink peer memory) and consumers wait on the producers'
    events; "nccl": grouped ncclSend / ncclRecv (needs distinct devices)."""

    def __init__(self, n_workers: int, devices=None, exchange: str = "peer"):
        self._h = C.c_void_p()
        mode = {"peer": _lib.SHTC_EXCHANGE_PEER, "nccl": _lib.SHTC_EXCHANGE_NCCL}[exchange]
        d = None if devices is None else np.ascontiguousarray(devices, np.int32)
        check(lib().shtc_group_create(int(n_workers), _p(d), mode, C.byref(self._h)), group=None)
        self.n_workers = n_workers
        self.exchange = exchange
        self.grid = None
        self.lmax = self.mmax = None

    def _check(self, rc):
        check(rc, group=self._h)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().shtc_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device(self, worker: int) -> int:
        d = C.c_int()
        self._check(lib().shtc_group_device(self._h, worker, C.byref(d)))
        return d.value

    def set_grid(self, grid: PixelGrid, mirror: bool = True):
        self._check(lib().shtc_group_set_grid(self._h, grid.n_rings, _p(grid.cos_theta), _p(grid.n_phi),
                                              _p(grid.phi_0), _p(grid.weight), _p(grid.pixel_offset),
                                              int(bool(mirror))))
        self.grid = grid

    def set_layout(self, lmax: int, mmax: int, m_sets, ring_sets):
        mo = np.full(mmax + 1, -1, np.int32)
        ro = np.full(self.grid.n_rings, -1, np.int32)
        for w, ms in enumerate(m_sets):
            mo[np.asarray(ms, np.int64)] = w
        for w, rs in enumerate(ring_sets):
            ro[np.asarray(rs, np.int64)] = w
        self._check(lib().shtc_group_set_layout(self._h, lmax, mmax, _p(mo), _p(ro)))
        self.lmax, self.mmax = lmax, mmax

    def plan_ms(self) -> float:
        t = C.c_double()
        self._check(lib().shtc_group_plan_ms(self._h, C.byref(t)))
        return t.value

    def alm2map(self, alm, out=None, timing=False):
        alm = np.ascontiguousarray(alm, np.complex128)
        if alm.size != alm_count(self.lmax, self.mmax):
            raise ValueError("alm2map: coefficient count != AlmSet::count(lmax, mmax)")
        mp = out if out is not None else np.empty(self.grid.n_pix)
        t = GroupTiming()
        self._check(lib().shtc_group_alm2map(self._h, _p(alm), _p(mp), C.byref(t)))
        return (mp, t.as_dict()) if timing else mp

    def map2alm(self, mp, out=None, timing=False):
        mp = np.ascontiguousarray(mp, np.float64)
        if mp.size != self.grid.n_pix:
            raise ValueError("analysis: pixel count != grid")
        alm = out if out is not None else np.empty(alm_count(self.lmax, self.mmax), np.complex128)
        t = GroupTiming()
        self._check(lib().shtc_group_map2alm(self._h, _p(mp), _p(alm), C.byref(t)))
        return (alm, t.as_dict()) if timing else alm

    def alm2map_dev(self, alm_ptrs, map_ptrs):
        """Per-worker device buffers (full triangle / full map on each worker's device)."""
        a = np.ascontiguousarray(alm_ptrs, np.uint64)
        m = np.ascontiguousarray(map_ptrs, np.uint64)
        t = GroupTiming()
        self._check(lib().shtc_group_alm2map_dev(self._h, _p(a), _p(m), C.byref(t)))
        return t.as_dict()

    def map2alm_dev(self, map_ptrs, alm_ptrs):
        m = np.ascontiguousarray(map_ptrs, np.uint64)
        a = np.ascontiguousarray(alm_ptrs, np.uint64)
        t = GroupTiming()
        self._check(lib().shtc_group_map2alm_dev(self._h, _p(m), _p(a), C.byref(t)))
        return t.as_dict()


def default_context(device: int = 0) -> Context:
    """Process-wide context per device (the reference API has no handle)."""
    if device not in _DEFAULT:
        _DEFAULT[device] = Context(device)
    return _DEFAULT[device]


def _grid_ctx(grid: PixelGrid, lmax: int, mmax: int, pairing: bool, device: int) -> Context:
    ctx = default_context(device)
    key = (id(grid), grid.n_rings, grid.n_pix, bool(pairing))
    if getattr(ctx, "_grid_key", None) != key:
        ctx.set_grid(grid, mirror=pairing)
        ctx._grid_key = key
        ctx._band_key = None
    if getattr(ctx, "_band_key", None) != (lmax, mmax):
        ctx.set_band(lmax, mmax)
        ctx._band_key = (lmax, mmax)
    return ctx


# ----------------------------------------------------------------------------------------
# reference-named operators
# ----------------------------------------------------------------------------------------
def synthesis(alm: np.ndarray, lmax: int, mmax: int, grid: PixelGrid, pairing: bool = True,
              device: int = 0) -> np.ndarray:
    """alm2map (transforms.cpp:402-445); mirror pairing is used whenever the grid allows it."""
    if grid.n_rings == 0:
        raise ValueError("synthesis: empty grid")
    return _grid_ctx(grid, lmax, mmax, pairing, device).alm2map(alm)


def analysis(mp: np.ndarray, lmax: int, mmax: int, grid: PixelGrid, pairing: bool = True,
             device: int = 0) -> np.ndarray:
    """map2alm (transforms.cpp:447-485)."""
    if lmax < mmax or mmax < 0:
        raise ValueError("analysis: need lmax >= mmax >= 0")
    if grid.n_rings == 0:
        raise ValueError("analysis: empty grid")
    if np.asarray(mp).size != grid.n_pix:
        raise ValueError("analysis: pixel count != grid")
    return _grid_ctx(grid, lmax, mmax, pairing, device).map2alm(mp)


def _checked_m_set(m_set, mmax, where):
    ms = sorted(int(m) for m in m_set)
    for i, m in enumerate(ms):
        if m < 0 or m > mmax:
            raise ValueError(f"{where}: order outside [0, mmax]")
        if i and ms[i - 1] == m:
            raise ValueError(f"{where}: duplicate order")
    return ms


def compute_delta_a(alm, lmax: int, mmax: int, cos_thetas, m_set, device: int = 0):
    """Delta panel [ring][m] (transforms.cpp:269-286); returns (panel, steps)."""
    ms = _checked_m_set(m_set, mmax, "compute_delta_a")
    x = np.ascontiguousarray(cos_thetas, np.float64)
    if np.any(~(np.abs(x) <= 1.0)):
        raise ValueError("compute_delta_a: cos_theta outside [-1, 1]")
    return default_context(device).delta_a(alm, lmax, mmax, x, ms)


def compute_delta_a_ring_major(alm, lmax, mmax, cos_thetas, m_set, n_work_items: int = 1, device: int = 0):
    """Same numbers as compute_delta_a (transforms.cpp:288-331): the loop order is a CPU detail."""
    if n_work_items < 1:
        raise ValueError("compute_delta_a_ring_major: n_work_items must be >= 1")
    ms = _checked_m_set(m_set, mmax, "compute_delta_a_ring_major")
    x = np.ascontiguousarray(cos_thetas, np.float64)
    if np.any(~(np.abs(x) <= 1.0)):
        raise ValueError("compute_delta_a_ring_major: cos_theta outside [-1, 1]")
    return default_context(device).delta_a(alm, lmax, mmax, x, ms)


def accumulate_alm(panel, rings, ms, cos_thetas, lmax: int, mmax: int, device: int = 0):
    """a_lm = sum_r Delta^S_m(r) P_lm (transforms.cpp:357-365); returns (alm, steps)."""
    rings = list(rings)
    if rings != list(range(len(rings))):
        raise ValueError("accumulate_alm: ring coverage incomplete")
    return _accumulate_core(panel, rings, ms, cos_thetas, lmax, mmax, "accumulate_alm", device)


def _accumulate_core(panel, rings, ms, cos_thetas, lmax, mmax, where, device):
    if lmax < mmax or mmax < 0:
        raise ValueError(f"{where}: need lmax >= mmax >= 0")
    x = np.ascontiguousarray(cos_thetas, np.float64)
    if len(x) != len(rings):
        raise ValueError(f"{where}: latitude count != panel rings")
    if np.any(~(np.abs(x) <= 1.0)):
        raise ValueError(f"{where}: cos_theta outside [-1, 1]")
    ms = [int(m) for m in ms]
    for m in ms:
        if m < 0 or m > mmax:
            raise ValueError(f"{where}: panel order outside [0, mmax]")
    panel = np.ascontiguousarray(panel, np.complex128).reshape(len(x), len(ms))
    order = np.argsort(ms, kind="stable")
    return default_context(device).accumulate_alm(panel[:, order], x, np.asarray(ms)[order], lmax, mmax)


@dataclass
class PartialAlm:
    alm: np.ndarray
    rings: list
    lmax: int
    mmax: int


def accumulate_alm_partial(panel, rings, ms, cos_thetas, lmax, mmax, device: int = 0):
    """transforms.cpp:367-378."""
    rings = list(rings)
    for i in range(1, len(rings)):
        if rings[i] <= rings[i - 1]:
            raise ValueError("accumulate_alm_partial: rings not strictly ascending")
    alm, steps = _accumulate_core(panel, rings, ms, cos_thetas, lmax, mmax, "accumulate_alm_partial", device)
    return PartialAlm(alm, rings, lmax, mmax), steps


def reduce_partials(parts, n_rings: int) -> np.ndarray:
    """Sums partials in list order after the disjoint/cover checks (transforms.cpp:380-400)."""
    if not parts:
        raise ValueError("reduce_partials: no partials")
    lmax, mmax = parts[0].lmax, parts[0].mmax
    seen = []
    for p in parts:
        if p.lmax != lmax or p.mmax != mmax:
            raise ValueError("reduce_partials: mismatched band limits")
        seen += list(p.rings)
    seen.sort()
    for i in range(1, len(seen)):
        if seen[i] == seen[i - 1]:
            raise ValueError("reduce_partials: overlapping ring subsets")
    if len(seen) != n_rings or (n_rings > 0 and (seen[0] != 0 or seen[-1] != n_rings - 1)):
        raise ValueError("reduce_partials: ring subsets do not cover the grid")
    out = np.zeros(alm_count(lmax, mmax), np.complex128)
    for p in parts:
        out += p.alm
    return out


def kernel_launches() -> int:
    """Kernel launches the library has issued in this process (shtc_kernel_launches)."""
    return int(lib().shtc_kernel_launches())


def device_count() -> int:
    return int(lib().shtc_device_count())


def device_info(device: int = 0):
    name = C.create_string_buffer(128)
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    check(lib().shtc_device_info(device, name, 128, C.byref(sm), C.byref(ma), C.byref(mi)))
    return {"name": name.value.decode(), "sm_count": sm.value, "cc": f"{ma.value}.{mi.value}"}


def measure_fp64_peak(device: int = 0):
    t, mhz = C.c_double(), C.c_double()
    check(lib().shtc_measure_fp64_peak(device, C.byref(t), C.byref(mhz)))
    return t.value, mhz.value
