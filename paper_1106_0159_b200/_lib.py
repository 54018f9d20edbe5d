"""ctypes binding of libshtc.so (the C ABI declared in include/shtc.h).

The library is built in-tree by `python -m paper_1106_0159_b200.build` (or
`__graft_entry__.build()`).  Loading fails loudly if it is missing: there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SHTC_VARIANT_LIB"]) if os.environ.get("SHTC_VARIANT_LIB") else PKG / "libshtc.so"  # variant: tuning experiments only

SHTC_OK, SHTC_EINVAL, SHTC_EDOMAIN, SHTC_ECUDA, SHTC_ENOMEM, SHTC_EUNSUPPORTED = range(6)

# every symbol include/shtc.h declares (checked by the CPU test suite)
EXPORTED = [
    "shtc_create", "shtc_destroy", "shtc_last_error", "shtc_device_count", "shtc_set_stream",
    "shtc_set_grid", "shtc_set_band", "shtc_plan", "shtc_plan_stats", "shtc_plan_phase_stats", "shtc_plan_executed", "shtc_alm2map",
    "shtc_map2alm", "shtc_alm2map_dev", "shtc_map2alm_dev", "shtc_set_exchange_layout",
    "shtc_set_exchange_layout_synthesis",
    "shtc_legendre_alm2map_dev", "shtc_legendre_map2alm_dev", "shtc_ring_synthesis_dev",
    "shtc_ring_analysis_dev", "shtc_delta_a", "shtc_accumulate_alm", "shtc_device_info",
    "shtc_measure_fp64_peak", "shtc_dev_alloc", "shtc_dev_free", "shtc_ipc_handle", "shtc_ipc_open",
    "shtc_ipc_close", "shtc_set_exchange_peers", "shtc_legendre_alm2map_peer", "shtc_ring_analysis_peer",
    "shtc_peer_barrier", "shtc_kernel_launches", "shtc_copy_orders", "shtc_host_alloc", "shtc_host_free",
    "shtc_group_create", "shtc_group_destroy", "shtc_group_last_error", "shtc_group_device",
    "shtc_group_set_grid", "shtc_group_set_layout", "shtc_group_plan_ms", "shtc_group_alm2map",
    "shtc_group_map2alm", "shtc_group_alm2map_dev", "shtc_group_map2alm_dev", "shtc_set_ladder",
]

SHTC_EXCHANGE_PEER, SHTC_EXCHANGE_NCCL = 0, 1


class Timing(C.Structure):
    _fields_ = [
        ("legendre_ms", C.c_double), ("fft_ms", C.c_double), ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double), ("total_ms", C.c_double), ("nominal_steps", C.c_uint64),
        ("executed_steps", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GroupTiming(C.Structure):
    _fields_ = [
        ("legendre_ms", C.c_double), ("fft_ms", C.c_double), ("exchange_ms", C.c_double),
        ("h2d_ms", C.c_double), ("d2h_ms", C.c_double), ("total_ms", C.c_double),
        ("exchange_bytes", C.c_uint64), ("nominal_steps", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_1106_0159_b200.build); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
        u64p = C.POINTER(C.c_uint64)
        L.shtc_last_error.restype = C.c_char_p
        L.shtc_last_error.argtypes = [vp]
        L.shtc_create.argtypes = [i32, C.POINTER(vp)]
        L.shtc_destroy.argtypes = [vp]
        L.shtc_destroy.restype = None
        L.shtc_device_count.restype = i32
        L.shtc_kernel_launches.restype = C.c_uint64
        L.shtc_kernel_launches.argtypes = []
        L.shtc_copy_orders.argtypes = [vp, vp, vp, i32]
        L.shtc_set_stream.argtypes = [vp, vp]
        L.shtc_set_grid.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32]
        L.shtc_set_band.argtypes = [vp, i32, i32, i32, vp]
        L.shtc_set_ladder.argtypes = [vp, i32]
        L.shtc_plan.argtypes = [vp, C.POINTER(dbl)]
        L.shtc_plan_stats.argtypes = [vp, u64p, u64p, u64p]
        L.shtc_plan_phase_stats.argtypes = [vp, u64p, u64p, u64p]
        L.shtc_plan_executed.argtypes = [vp, u64p, u64p]
        for f in ("shtc_alm2map", "shtc_map2alm", "shtc_alm2map_dev", "shtc_map2alm_dev",
                  "shtc_legendre_alm2map_dev", "shtc_legendre_map2alm_dev",
                  "shtc_ring_synthesis_dev", "shtc_ring_analysis_dev"):
            getattr(L, f).argtypes = [vp, vp, vp, C.POINTER(Timing)]
        L.shtc_set_exchange_layout.argtypes = [vp, vp, i32, vp, vp, vp]
        L.shtc_set_exchange_layout_synthesis.argtypes = [vp, vp, vp, vp, vp]
        L.shtc_delta_a.argtypes = [vp, vp, i32, i32, i32, vp, i32, vp, vp, u64p]
        L.shtc_accumulate_alm.argtypes = [vp, vp, i32, vp, i32, vp, i32, i32, vp, u64p]
        L.shtc_device_info.argtypes = [i32, C.c_char_p, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.shtc_measure_fp64_peak.argtypes = [i32, C.POINTER(dbl), C.POINTER(dbl)]
        L.shtc_dev_alloc.argtypes = [i32, C.c_uint64, C.POINTER(vp)]
        L.shtc_dev_free.argtypes = [vp]
        L.shtc_ipc_handle.argtypes = [vp, C.c_char_p]
        L.shtc_ipc_open.argtypes = [i32, C.c_char_p, C.POINTER(vp)]
        L.shtc_ipc_close.argtypes = [vp]
        L.shtc_set_exchange_peers.argtypes = [vp, vp, vp]
        L.shtc_legendre_alm2map_peer.argtypes = [vp, vp, C.POINTER(Timing)]
        L.shtc_ring_analysis_peer.argtypes = [vp, vp, C.POINTER(Timing)]
        L.shtc_peer_barrier.argtypes = [vp, i32, i32, vp, C.c_uint32]
        L.shtc_group_create.argtypes = [i32, vp, i32, C.POINTER(vp)]
        L.shtc_group_destroy.argtypes = [vp]
        L.shtc_group_destroy.restype = None
        L.shtc_group_last_error.argtypes = [vp]
        L.shtc_group_last_error.restype = C.c_char_p
        L.shtc_group_device.argtypes = [vp, i32, C.POINTER(i32)]
        L.shtc_group_set_grid.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32]
        L.shtc_group_set_layout.argtypes = [vp, i32, i32, vp, vp]
        L.shtc_group_plan_ms.argtypes = [vp, C.POINTER(dbl)]
        for f in ("shtc_group_alm2map", "shtc_group_map2alm", "shtc_group_alm2map_dev", "shtc_group_map2alm_dev"):
            getattr(L, f).argtypes = [vp, vp, vp, C.POINTER(GroupTiming)]
        _LIB = L
    return _LIB


class ShtcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc: int, ctx=None, group=None):
    if rc == SHTC_OK:
        return
    msg = (lib().shtc_group_last_error(group) if group is not None else lib().shtc_last_error(ctx)).decode(errors="replace")
    # error classes of the reference (std::invalid_argument / std::domain_error)
    if rc == SHTC_EINVAL:
        raise ValueError(msg)
    if rc == SHTC_EDOMAIN:
        raise ArithmeticError(msg)
    if rc == SHTC_ENOMEM:
        raise MemoryError(msg)
    raise ShtcError(rc, msg)
