"""Measured exchange parameters for the perfmodel (sht::CostParams::b200, sht::fit_exchange).

alpha (fused path): the per-exchange fixed cost of the fused peer-store exchange is one
device-side barrier (shtc_peer_barrier) -- W single-thread kernels publishing an epoch and
spinning on the others' flags.  Timed here for W workers of one process on device 0, K
barrier rounds back to back (device-wide synchronisation around the loop).

beta: the fused path's bytes ride inside the producing kernels; with more than one GPU the
script times peer copies (tensor.to(other device)) over a size sweep and fits
t = a + s / bw.  With one GPU there is no NVLink to measure, so beta stays the B200
profiling guide's measured peer figure and the output says so.

    python tools/calibrate_exchange.py > profiles/r02_exchange_calibration.json
"""
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("SHTC_FFT_AUX", "2")
sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import sht


def barrier_latency(W, rounds=200):
    grid = sht.build_healpix_grid(8)
    lmax = 16
    layout = sht.WorkerLayout.create(grid, lmax, W)
    peers = [None] * W
    xs = []
    for w in range(W):
        c = sht.Context(0)
        c.set_grid(grid)
        c.set_band(lmax, lmax, layout.m_sets[w])
        xs.append(sht.PeerExchange(c, layout, w, peers=peers))
    for x in xs:
        x.connect()
    for _ in range(10):
        for x in xs:
            x.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(rounds):
        for x in xs:
            x.barrier()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / rounds
    for x in xs:
        x.close()
    return dt


def peer_copy_fit(n_dev):
    if n_dev < 2:
        return None
    sizes = [1 << k for k in range(16, 29, 2)]
    ts = []
    for s in sizes:
        a = torch.empty(s // 8, dtype=torch.float64, device="cuda:0")
        b = a.to("cuda:1")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            b.copy_(a, non_blocking=True)
        torch.cuda.synchronize("cuda:0")
        torch.cuda.synchronize("cuda:1")
        ts.append((time.perf_counter() - t0) / 10)
    A = np.stack([np.ones(len(sizes)), np.array(sizes, float)], 1)
    (alpha, beta), *_ = np.linalg.lstsq(A, np.array(ts), rcond=None)
    return {"alpha_s": float(alpha), "beta_inv_bw_s_per_byte": float(beta), "bw_gbs": 1e-9 / float(beta),
            "samples": [[s, t] for s, t in zip(sizes, ts)]}


def main():
    n_dev = sht.device_count()
    out = {"device": torch.cuda.get_device_name(0), "n_devices": n_dev,
           "barrier_s": {str(W): barrier_latency(W) for W in (2, 4, 8)}}
    fit = peer_copy_fit(n_dev)
    out["peer_copy_fit"] = fit if fit else ("one GPU: no NVLink peer link to time; beta stays the "
                                            "B200 profiling guide's measured 770 GB/s per direction")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
