"""Fused-exchange store coalescing on one GPU: W workers of one process on device 0 run the
peer-store stages (Legendre alm2map -> receive blocks, ring analysis -> send blocks) with the
order-major synthesis blocks (default) or the ring-major ones (--ring-major), so ncu can count
the store sectors per request of the two producing kernels:

    CUDA_DEVICE_MAX_CONNECTIONS=32 SHTC_FFT_AUX=2 ncu --metrics \\
        l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum \\
        -k regex:"leg_alm2map_kernel|ring_p2_anal" python tools/exchange_coalesce.py --stage-only [--ring-major]

Without ncu it prints the per-stage times of both layouts (stage kernels only, the barrier
excluded)."""
import argparse
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("SHTC_FFT_AUX", "2")
sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import sht


def run(nside, lmax, W, order_major, reps, stage_only=False):
    dev = torch.device("cuda", 0)
    grid = sht.build_healpix_grid(nside)
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
    alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 12345).view(np.float64)).to(dev)
    mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
    out = torch.zeros_like(alm)
    if stage_only:  # the two peer-store kernels alone (no barrier: ncu serialises kernels)
        for x in xs:
            x.ctx.legendre_alm2map_peer(alm.data_ptr())
        for x in xs:
            x.ctx.ring_analysis_peer(mp.data_ptr())
        torch.cuda.synchronize()
        for x in xs:
            x.close()
        return
    leg, anal = [], []
    for _ in range(reps):
        # stage by stage (a timed call synchronises; a barrier must not be waited on before
        # every worker has reached it)
        tl = sum(x.ctx.legendre_alm2map_peer(alm.data_ptr(), True)["legendre_ms"] for x in xs)
        for x in xs:
            x.barrier()
            x.ctx.ring_synthesis_dev(x.recv, mp.data_ptr())
        torch.cuda.synchronize()
        ta = sum(x.ctx.ring_analysis_peer(mp.data_ptr(), True)["fft_ms"] for x in xs)
        for x in xs:
            x.barrier()
            x.ctx.legendre_map2alm_dev(x.send, out.data_ptr())
        torch.cuda.synchronize()
        leg.append(tl)
        anal.append(ta)
    torch.cuda.synchronize()
    for x in xs:
        x.close()
    tag = "order-major" if order_major else "ring-major"
    print(f"{tag:12s} W={W} nside={nside} lmax={lmax}: Legendre alm2map (peer stores) {min(leg):.3f} ms, "
          f"ring analysis (peer stores) {min(anal):.3f} ms (sum over workers, best of {reps})", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--nside", type=int, default=1024)
    ap.add_argument("--lmax", type=int, default=2048)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ring-major", action="store_true")
    ap.add_argument("--both", action="store_true")
    ap.add_argument("--stage-only", action="store_true")
    a = ap.parse_args()
    if a.both:
        run(a.nside, a.lmax, a.workers, True, a.reps)
        run(a.nside, a.lmax, a.workers, False, a.reps)
    else:
        run(a.nside, a.lmax, a.workers, not a.ring_major, a.reps, a.stage_only)
