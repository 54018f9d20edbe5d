"""TEST INFRASTRUCTURE ONLY — ctypes binding of the reference implementation.

`oracle/_ref/libsht_ref.so` is the UNMODIFIED reference (/root/reference/proj/src/*.cpp)
compiled by `oracle/build_ref.sh` plus the C shim `oracle/ref_shim.cpp`.  Only tests/,
bench.py (cpu_baseline and --impl reference) and __graft_entry__.smoke() import this module,
and only as the checker / CPU baseline.  The product path never loads it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libsht_ref.so"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = C.POINTER(C.c_uint64)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


_LIB = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run oracle/build_ref.sh")
        L = C.CDLL(str(LIB_PATH))
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix64_at.restype = C.c_uint64
        L.ref_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_uniform_pm1.restype = C.c_double
        L.ref_uniform_pm1.argtypes = [C.c_uint64, C.c_uint64]
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


# ---- grids -----------------------------------------------------------------------------
class Grid:
    """Plain-array mirror of sht::PixelGrid (grid.hpp:27-37)."""

    def __init__(self, scheme, nside, cos_theta, n_phi, phi_0, weight):
        self.scheme = scheme  # 0 healpix, 1 gauss-legendre
        self.nside = nside
        self.cos_theta = np.ascontiguousarray(cos_theta, dtype=np.float64)
        self.n_phi = np.ascontiguousarray(n_phi, dtype=np.int32)
        self.phi_0 = np.ascontiguousarray(phi_0, dtype=np.float64)
        self.weight = np.ascontiguousarray(weight, dtype=np.float64)
        self.pixel_offset = np.concatenate([[0], np.cumsum(self.n_phi.astype(np.int64))[:-1]]).astype(np.int64)
        self.n_pix = int(self.n_phi.astype(np.int64).sum())

    @property
    def n_rings(self):
        return len(self.cos_theta)

    def args(self):
        return (self.scheme, self.nside, self.n_rings, self.cos_theta, self.n_phi, self.phi_0,
                self.weight)


def healpix_grid(nside: int) -> Grid:
    n = 4 * nside - 1
    z = np.zeros(n); nphi = np.zeros(n, np.int32); p0 = np.zeros(n); w = np.zeros(n)
    off = np.zeros(n, np.int64)
    _check(lib().ref_healpix_grid(C.c_int(nside), z.ctypes.data_as(C.c_void_p),
                                  nphi.ctypes.data_as(C.c_void_p), p0.ctypes.data_as(C.c_void_p),
                                  w.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p)))
    return Grid(0, nside, z, nphi, p0, w)


def gl_grid(n_rings: int, n_phi: int) -> Grid:
    z = np.zeros(n_rings); nphi = np.zeros(n_rings, np.int32); p0 = np.zeros(n_rings)
    w = np.zeros(n_rings); off = np.zeros(n_rings, np.int64)
    _check(lib().ref_gl_grid(C.c_int(n_rings), C.c_int(n_phi), z.ctypes.data_as(C.c_void_p),
                             nphi.ctypes.data_as(C.c_void_p), p0.ctypes.data_as(C.c_void_p),
                             w.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p)))
    return Grid(1, 0, z, nphi, p0, w)


def gl_nodes(n: int):
    x = np.zeros(n); w = np.zeros(n)
    _check(lib().ref_gl_nodes(C.c_int(n), x.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))
    return x, w


# ---- legendre ----------------------------------------------------------------------------
def log_mu(m: int) -> float:
    out = C.c_double()
    _check(lib().ref_log_mu(C.c_int(m), C.byref(out)))
    return out.value


def beta_lm(l: int, m: int) -> float:
    out = C.c_double()
    _check(lib().ref_beta_lm(C.c_int(l), C.c_int(m), C.byref(out)))
    return out.value


def pmm_from_log(m: int, x: float, lmu: float):
    mant = C.c_double(); sc = C.c_int32()
    _check(lib().ref_pmm_from_log(C.c_int(m), C.c_double(x), C.c_double(lmu), C.byref(mant), C.byref(sc)))
    return mant.value, sc.value


def plm_row(m: int, x: float, lmax: int, unscaled: bool = False) -> np.ndarray:
    out = np.zeros(max(lmax - m + 1, 0))
    _check(lib().ref_plm_row(C.c_int(m), C.c_double(x), C.c_int(lmax), C.c_int(int(unscaled)),
                             out.ctypes.data_as(C.c_void_p)))
    return out


def plm_row_scaled(m: int, x: float, lmax: int):
    mant = np.zeros(lmax - m + 1); sc = np.zeros(lmax - m + 1, np.int32)
    _check(lib().ref_plm_row_scaled(C.c_int(m), C.c_double(x), C.c_int(lmax),
                                    mant.ctypes.data_as(C.c_void_p), sc.ctypes.data_as(C.c_void_p)))
    return mant, sc


# ---- inputs ------------------------------------------------------------------------------
def alm_count(lmax: int, mmax: int) -> int:
    return (mmax + 1) * (lmax + 1) - mmax * (mmax + 1) // 2


def splitmix64_at(seed: int, index: int) -> int:
    return int(lib().ref_splitmix64_at(seed, index))


def random_alm(lmax: int, mmax: int, seed: int) -> np.ndarray:
    out = np.zeros(2 * alm_count(lmax, mmax))
    _check(lib().ref_random_alm(C.c_int(lmax), C.c_int(mmax), C.c_uint64(seed),
                                out.ctypes.data_as(C.c_void_p)))
    return out.view(np.complex128)


# ---- transforms ----------------------------------------------------------------------------
def _gridargs(g: Grid):
    return (C.c_int(g.scheme), C.c_int(g.nside), C.c_int(g.n_rings),
            g.cos_theta.ctypes.data_as(C.c_void_p), g.n_phi.ctypes.data_as(C.c_void_p),
            g.phi_0.ctypes.data_as(C.c_void_p), g.weight.ctypes.data_as(C.c_void_p))


def synthesis(alm: np.ndarray, lmax: int, mmax: int, g: Grid, pairing=True, ring_major=False):
    a = np.ascontiguousarray(alm, dtype=np.complex128)
    out = np.zeros(g.n_pix)
    steps = C.c_uint64(0)
    _check(lib().ref_synthesis(C.c_int(lmax), C.c_int(mmax), a.ctypes.data_as(C.c_void_p), *_gridargs(g),
                               C.c_int(int(pairing)), C.c_int(int(ring_major)),
                               out.ctypes.data_as(C.c_void_p), C.byref(steps)))
    return out, steps.value


def analysis(mp: np.ndarray, lmax: int, mmax: int, g: Grid, pairing=True):
    m = np.ascontiguousarray(mp, dtype=np.float64)
    out = np.zeros(2 * alm_count(lmax, mmax))
    steps = C.c_uint64(0)
    _check(lib().ref_analysis(C.c_int(lmax), C.c_int(mmax), m.ctypes.data_as(C.c_void_p), *_gridargs(g),
                              C.c_int(int(pairing)), out.ctypes.data_as(C.c_void_p), C.byref(steps)))
    return out.view(np.complex128), steps.value


def compute_delta_a(alm, lmax, mmax, x, ms, ring_major=False, n_work_items=1, unscaled=False):
    a = np.ascontiguousarray(alm, dtype=np.complex128)
    x = np.ascontiguousarray(x, dtype=np.float64)
    ms = np.ascontiguousarray(ms, dtype=np.int32)
    out = np.zeros((len(x), len(ms)), np.complex128)
    steps = C.c_uint64(0)
    _check(lib().ref_compute_delta_a(C.c_int(lmax), C.c_int(mmax), a.ctypes.data_as(C.c_void_p),
                                     C.c_int(len(x)), x.ctypes.data_as(C.c_void_p), C.c_int(len(ms)),
                                     ms.ctypes.data_as(C.c_void_p), C.c_int(int(ring_major)),
                                     C.c_int(n_work_items), C.c_int(int(unscaled)),
                                     out.ctypes.data_as(C.c_void_p), C.byref(steps)))
    return out, steps.value


def accumulate_alm(delta, x, ms, lmax, mmax):
    d = np.ascontiguousarray(delta, dtype=np.complex128)
    x = np.ascontiguousarray(x, dtype=np.float64)
    ms = np.ascontiguousarray(ms, dtype=np.int32)
    out = np.zeros(2 * alm_count(lmax, mmax))
    steps = C.c_uint64(0)
    _check(lib().ref_accumulate_alm(C.c_int(lmax), C.c_int(mmax), C.c_int(len(x)), x.ctypes.data_as(C.c_void_p),
                                    C.c_int(len(ms)), ms.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
                                    out.ctypes.data_as(C.c_void_p), C.byref(steps)))
    return out.view(np.complex128), steps.value


def ring_synthesis(delta, n_phi, phi_0):
    d = np.ascontiguousarray(delta, dtype=np.complex128)
    out = np.zeros(n_phi)
    _check(lib().ref_ring_synthesis(C.c_int(len(d)), d.ctypes.data_as(C.c_void_p), C.c_int(n_phi),
                                    C.c_double(phi_0), out.ctypes.data_as(C.c_void_p)))
    return out


def ring_analysis(samples, phi_0, weight, mmax):
    s = np.ascontiguousarray(samples, dtype=np.float64)
    out = np.zeros(mmax + 1, np.complex128)
    _check(lib().ref_ring_analysis(C.c_int(len(s)), s.ctypes.data_as(C.c_void_p), C.c_double(phi_0),
                                   C.c_double(weight), C.c_int(mmax), out.ctypes.data_as(C.c_void_p)))
    return out


def _sets(fn, n_sets, total, *args):
    counts = np.zeros(n_sets, np.int32)
    flat = np.zeros(max(total, 1), np.int32)
    _check(fn(*args, counts.ctypes.data_as(C.c_void_p), flat.ctypes.data_as(C.c_void_p)))
    out, k = [], 0
    for c in counts:
        out.append([int(v) for v in flat[k:k + c]]); k += c
    return out


def assign_m(mmax: int, n_workers: int):
    return _sets(lib().ref_assign_m, n_workers, mmax + 1, C.c_int(mmax), C.c_int(n_workers))


def assign_rings_healpix(nside: int, n_workers: int):
    return _sets(lib().ref_assign_rings_healpix, n_workers, 4 * nside - 1, C.c_int(nside), C.c_int(n_workers))


def thread_partition(ms, n_threads):
    a = np.ascontiguousarray(ms, dtype=np.int32)
    return _sets(lib().ref_thread_partition, n_threads, len(a), C.c_int(len(a)), a.ctypes.data_as(C.c_void_p),
                 C.c_int(n_threads))


def distributed_synthesis(alm, lmax, mmax, g: Grid, n_workers=1, n_threads=1, pairing=True, ring_major=False):
    a = np.ascontiguousarray(alm, dtype=np.complex128)
    out = np.zeros(g.n_pix)
    st = np.zeros(4)
    tot = np.zeros(2, np.uint64)
    _check(lib().ref_distributed_synthesis(C.c_int(lmax), C.c_int(mmax), a.ctypes.data_as(C.c_void_p),
                                           *_gridargs(g), C.c_int(n_workers), C.c_int(n_threads),
                                           C.c_int(int(pairing)), C.c_int(int(ring_major)),
                                           out.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                                           tot.ctypes.data_as(C.c_void_p)))
    return out, {"precompute_s": st[0], "recurrence_s": st[1], "exchange_s": st[2], "fft_s": st[3],
                 "exchange_bytes": int(tot[0]), "steps": int(tot[1])}


def distributed_analysis(mp, lmax, mmax, g: Grid, n_workers=1, n_threads=1, pairing=True, ring_major=False):
    m = np.ascontiguousarray(mp, dtype=np.float64)
    out = np.zeros(2 * alm_count(lmax, mmax))
    st = np.zeros(4)
    tot = np.zeros(2, np.uint64)
    _check(lib().ref_distributed_analysis(C.c_int(lmax), C.c_int(mmax), m.ctypes.data_as(C.c_void_p),
                                          *_gridargs(g), C.c_int(n_workers), C.c_int(n_threads),
                                          C.c_int(int(pairing)), C.c_int(int(ring_major)),
                                          out.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                                          tot.ctypes.data_as(C.c_void_p)))
    return out.view(np.complex128), {"precompute_s": st[0], "recurrence_s": st[1], "exchange_s": st[2],
                                     "fft_s": st[3], "exchange_bytes": int(tot[0]), "steps": int(tot[1])}
