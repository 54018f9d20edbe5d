"""Per-rank compute of the W-GPU m-distributed step, timed on one GPU: each worker's
Legendre stages (its orders, every ring) and ring stages (its rings) on its share, the
exchange excluded.  max over ranks of the per-rank step time against the single-GPU step
gives the compute-only strong-scaling efficiency the W-GPU run can reach (the fused
exchange overlaps the Legendre epilogue; its barrier and NVLink time come on top).

    python tools/rank_share.py [nside lmax]     # prints one JSON line
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import sht

nside, lmax = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 4096)))
RINGS = sys.argv[4] if len(sys.argv) > 4 else "interleaved"
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)  # explicit: the library and the events share it
torch.cuda.set_stream(stream)
g = sht.build_healpix_grid(nside)
alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 12345).view(np.float64)).to(dev)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = {"config": f"HEALPix nside={nside} lmax=mmax={lmax}", "per_W": {}}
single = None
for W in (1, 2, 4, 8):
    layout = sht.WorkerLayout.create(g, lmax, W, rings=RINGS)
    per_rank = []
    for r in range(W):
        c = sht.Context(0)
        c.set_stream(stream.cuda_stream)
        c.set_grid(g)
        c.set_band(lmax, lmax, layout.m_sets[r])
        row_off, send_c, recv_c, ring_list, m_base, m_stride = sht.exchange_layout(layout, r)
        c.set_exchange_layout(row_off, ring_list, m_base, m_stride)
        c.plan()
        send = torch.zeros(2 * max(1, sum(send_c)), dtype=torch.float64, device=dev)
        recv = torch.zeros(2 * max(1, sum(recv_c)), dtype=torch.float64, device=dev)
        mp = torch.zeros(g.n_pix, dtype=torch.float64, device=dev)
        ao = torch.zeros_like(alm)

        def step():
            c.legendre_alm2map_dev(alm.data_ptr(), send.data_ptr())
            c.ring_synthesis_dev(recv.data_ptr(), mp.data_ptr())
            c.ring_analysis_dev(mp.data_ptr(), recv.data_ptr())
            c.legendre_map2alm_dev(send.data_ptr(), ao.data_ptr())
        per_rank.append(timed(step))
        if W == 8 or (len(sys.argv) > 3 and sys.argv[3] == "stages"):
            st = [c.legendre_alm2map_dev(alm.data_ptr(), send.data_ptr(), timing=True)["legendre_ms"],
                  c.ring_synthesis_dev(recv.data_ptr(), mp.data_ptr(), timing=True)["fft_ms"],
                  c.ring_analysis_dev(mp.data_ptr(), recv.data_ptr(), timing=True)["fft_ms"],
                  c.legendre_map2alm_dev(send.data_ptr(), ao.data_ptr(), timing=True)["legendre_ms"]]
            ps = c.plan_stats()
            print(f"  W={W} rank {r}: leg_a2m {st[0]:.3f} synth {st[1]:.3f} anal {st[2]:.3f} leg_m2a {st[3]:.3f} "
                  f"orders {len(layout.m_sets[r])} executed {ps['executed'] / 1e9:.3f}G", flush=True)
        c.close()
        del send, recv, mp, ao
        torch.cuda.empty_cache()
    t = max(per_rank)
    if W == 1:
        single = t
    out["per_W"][W] = {"ms_per_rank": [round(x, 3) for x in per_rank], "max_ms": round(t, 3),
                       "compute_only_efficiency": round(single / (W * t), 4)}
    print(W, out["per_W"][W], flush=True)
print(json.dumps(out))
