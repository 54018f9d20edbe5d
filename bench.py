#!/usr/bin/env python
"""Benchmark driver: alm2map + map2alm on HEALPix nside=2048, lmax=mmax=4096 (BASELINE C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one alm2map of a Gaussian a_lm followed by one map2alm of the resulting map
(both FP64, the paper's two transforms).  `value` = whole-job algorithmic FP64 TFLOP/s
(8 flops per (l, m, ring-pair) step of the reference's mirror path, both transforms,
SURVEY.md §8d) over the device-timed step (inputs already in HBM, max over ranks).
`e2e` runs the same step through the host-buffer C ABI (shtc_alm2map / shtc_map2alm) from
pinned host memory, host<->device copies inside the timed region.

N > 1 (torchrun, one process per GPU, NCCL): orders are dealt with the reference's
assign_m, rings with assign_rings; the Legendre stage writes the packed all-to-all send
buffer directly, one NCCL all-to-all moves Delta, the ring stage reads the receive buffer
directly (strong scaling: total work fixed).

--impl reference times the reference's own CPU implementation (oracle/_ref, built from
/root/reference by oracle/build_ref.sh) on the host cores, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "alm2map/map2alm ms & FP64 TFLOP/s, nside=2048 ℓmax=4096, 1/2/4/8 B200"
NSIDE, LMAX = 2048, 4096
SEED_ALM = 12345


def falg_flops(lmax: int, mmax: int, n_rings: int) -> float:
    """F_alg = 8 x n_alm x ceil(R_N / 2) per transform."""
    n_alm = (mmax + 1) * (lmax + 1) - mmax * (mmax + 1) // 2
    return 8.0 * n_alm * ((n_rings + 1) // 2)


# ----------------------------------------------------------------------------------------
# clocks
# ----------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons}


# ----------------------------------------------------------------------------------------
# CPU baseline: the reference itself (oracle/_ref), bounded sample
# ----------------------------------------------------------------------------------------
def cpu_baseline(nside: int = NSIDE, lmax: int = LMAX, transforms=("alm2map", "map2alm")):
    """The reference's own CPU implementation (oracle/_ref: the unmodified sources compiled
    here) on the workload's own config: one alm2map and one map2alm of the bench's Gaussian
    a_lm, through distributed_synthesis / distributed_analysis (distribution.cpp:300-490) with
    1 worker x all host threads and PairPolicy::mirror, its fastest path.  No projection, no
    smaller stand-in grid: the same transforms the GPU step runs."""
    from oracle import ref
    from paper_1106_0159_b200 import sht
    threads = os.cpu_count() or 1
    g = ref.healpix_grid(nside)
    a = sht.gaussian_alm(lmax, lmax, SEED_ALM)
    out = {"unit": "TFLOP/s", "cores": threads, "kind": "reference"}
    fl = 0.0
    t_total = 0.0
    m = None
    if "alm2map" in transforms:
        t0 = time.perf_counter()
        m, st1 = ref.distributed_synthesis(a, lmax, lmax, g, 1, threads, pairing=True)
        dt = time.perf_counter() - t0
        out["ms_alm2map"] = dt * 1e3
        out["stages_alm2map_s"] = {k: st1[k] for k in ("recurrence_s", "fft_s", "exchange_s")}
        fl += falg_flops(lmax, lmax, g.n_rings)
        t_total += dt
    if "map2alm" in transforms:
        if m is None:
            m = sht.gaussian_map(int(g.n_pix), 2026)
        t0 = time.perf_counter()
        _, st2 = ref.distributed_analysis(m, lmax, lmax, g, 1, threads, pairing=True)
        dt = time.perf_counter() - t0
        out["ms_map2alm"] = dt * 1e3
        out["stages_map2alm_s"] = {k: st2[k] for k in ("recurrence_s", "fft_s", "exchange_s")}
        fl += falg_flops(lmax, lmax, g.n_rings)
        t_total += dt
    out["value"] = fl / t_total / 1e12
    out["ms_per_step"] = t_total * 1e3
    names = " + ".join(transforms)
    out["sample"] = (f"{names} at HEALPix nside={nside}, lmax=mmax={lmax} (the workload's own config, "
                     f"Gaussian a_lm seed {SEED_ALM}; map2alm of that alm2map output), reference "
                     f"distributed_synthesis/analysis, 1 worker x {threads} threads, PairPolicy::mirror")
    return out


# ----------------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def dist_ready():
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False


def config_tag(nside: int, lmax: int) -> str:
    """BASELINE.json config label of a (nside, lmax) pair."""
    tags = {(128, 256): " (C1)", (1024, 2048): " (C2/C3)", (2048, 4096): " (C4)", (4096, 8192): " (C5)"}
    return tags.get((nside, lmax), "")


def l2_note(n_alm: int, n_pix: int, n_rings: int, mmax: int) -> str:
    mb = lambda b: f"{b / 1e6:.0f} MB"  # noqa: E731
    sizes = (n_alm * 16, n_pix * 8, n_rings * (mmax + 1) * 16)
    rel = "larger than" if min(sizes) > 126e6 else "not all larger than"
    return f"inputs {rel} L2 (a_lm {mb(sizes[0])}, map {mb(sizes[1])}, Delta {mb(sizes[2])})"


def run_ours(args):
    import torch
    from paper_1106_0159_b200 import sht

    ws, rank, local = dist_env()
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"  # rank 0 prints exactly one JSON line on stdout
    # SHT_BENCH_SHARED_GPU=1 (testing the multi-rank path on one GPU): every rank on device 0,
    # gloo for the control plane (NCCL refuses two ranks on one device); the Delta exchange
    # is the peer-memory one, which needs no collective
    shared = os.environ.get("SHT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
        if args.exchange == "nccl":
            raise SystemExit("SHT_BENCH_SHARED_GPU=1 needs --exchange peer or none")
    backend = "gloo" if shared else "nccl"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group(backend, **({} if shared else {"device_id": dev}))
    grid = sht.build_healpix_grid(args.nside)
    lmax = mmax = args.lmax
    ctx = sht.Context(local)
    # one explicit stream shared by the library, torch (events, copies) and NCCL ordering; the
    # legacy default stream (handle 0) would fall back to the library's own stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    ctx.set_stream(stream.cuda_stream)
    ctx.set_grid(grid, mirror=True)

    alm_h = sht.gaussian_alm(lmax, mmax, SEED_ALM)
    n_alm = alm_h.size
    # ring sets of equal ring-stage cost (assign_rings_balanced); orders by the reference's
    # min-max pairs (assign_m): executed Legendre work balanced to 0.3% at 8 workers
    layout = sht.WorkerLayout.create(grid, mmax, ws, rings="balanced")
    Mi = layout.m_sets[rank]
    if args.exchange == "auto":
        args.exchange = "peer" if ws > 1 else "none"
    if ws == 1 and args.exchange == "none":
        ctx.set_band(lmax, mmax)
    else:
        ctx.set_band(lmax, mmax, Mi)
        if not dist_ready():
            import torch.distributed as dist
            if "RANK" not in os.environ:  # N=1 exchange path outside torchrun
                import socket
                so = socket.socket()
                so.bind(("127.0.0.1", 0))
                os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                                  MASTER_PORT=str(so.getsockname()[1]))
                so.close()
            dist.init_process_group(backend, **({} if shared else {"device_id": dev}))
    t0 = time.perf_counter()
    ctx.plan()
    plan_s = time.perf_counter() - t0
    stats = ctx.plan_stats()

    alm = torch.from_numpy(alm_h.view(np.float64)).to(dev)
    alm_out = torch.zeros_like(alm)
    launches_per_step = None
    exch_ms, exch_bytes = [], 0

    use_exchange = args.exchange != "none"
    # Every step records CUDA events on the shared stream between its stages (no host
    # synchronisation): [start, Legendre alm2map, (exchange), ring synthesis, ring analysis,
    # (exchange), Legendre map2alm].  The stage times of the timed steps come from them.
    mark = lambda evs, k: evs[k].record(stream) if evs is not None else None  # noqa: E731
    if not use_exchange:
        mp = torch.empty(grid.n_pix, dtype=torch.float64, device=dev)
        # the whole-transform kernels through the stage entry points (identity layout: the
        # same launches as shtc_alm2map_dev / shtc_map2alm_dev), Delta in its own buffer
        delta = torch.empty(2 * grid.n_rings * (mmax + 1), dtype=torch.float64, device=dev)
        n_marks = 5

        def step(evs=None):
            mark(evs, 0)
            ctx.legendre_alm2map_dev(alm.data_ptr(), delta.data_ptr())
            mark(evs, 1)
            ctx.ring_synthesis_dev(delta.data_ptr(), mp.data_ptr())
            mark(evs, 2)
            ctx.ring_analysis_dev(mp.data_ptr(), delta.data_ptr())
            mark(evs, 3)
            ctx.legendre_map2alm_dev(delta.data_ptr(), alm_out.data_ptr())
            mark(evs, 4)

        def stages(evs):  # legendre a2m, fft synth, fft anal, legendre m2a, exchange
            return (evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2]), evs[2].elapsed_time(evs[3]),
                    evs[3].elapsed_time(evs[4]), 0.0)
    elif args.exchange == "peer":
        # fused exchange: the Legendre (alm2map) and ring-analysis (map2alm) kernels store
        # Delta straight into the consumers' buffers over NVLink (CUDA IPC peer mappings),
        # then one device-side barrier; no collective on the data path
        import torch.distributed as dist

        def all_gather(obj):
            out = [None] * ws
            dist.all_gather_object(out, obj)
            return out
        px = sht.PeerExchange(ctx, layout, rank, all_gather=all_gather)
        send_c, recv_c = sht.exchange_sizes(layout, rank)
        mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
        _, sc, _, _, _, _ = sht.exchange_layout(layout, rank)
        exch_bytes = 16 * sum(c for j, c in enumerate(sc) if j != rank)
        n_marks = 7

        def step(evs=None):
            mark(evs, 0)
            ctx.legendre_alm2map_peer(alm.data_ptr())
            mark(evs, 1)
            px.barrier()
            mark(evs, 2)
            ctx.ring_synthesis_dev(px.recv, mp.data_ptr())
            mark(evs, 3)
            ctx.ring_analysis_peer(mp.data_ptr())
            mark(evs, 4)
            px.barrier()
            mark(evs, 5)
            ctx.legendre_map2alm_dev(px.send, alm_out.data_ptr())
            mark(evs, 6)

        def stages(evs):
            return (evs[0].elapsed_time(evs[1]), evs[2].elapsed_time(evs[3]), evs[3].elapsed_time(evs[4]),
                    evs[5].elapsed_time(evs[6]), evs[1].elapsed_time(evs[2]) + evs[4].elapsed_time(evs[5]))
    else:
        import torch.distributed as dist
        row_off, send_c, recv_c, ring_list, m_base, m_stride = sht.exchange_layout(layout, rank)
        ctx.set_exchange_layout(row_off, ring_list, m_base, m_stride)
        ctx.set_exchange_layout_synthesis(*sht.exchange_layout_synthesis(layout, rank))
        send = torch.empty(2 * sum(send_c), dtype=torch.float64, device=dev)
        recv = torch.empty(2 * sum(recv_c), dtype=torch.float64, device=dev)
        mp = torch.zeros(grid.n_pix, dtype=torch.float64, device=dev)
        s_split = [2 * c for c in send_c]
        r_split = [2 * c for c in recv_c]
        exch_bytes = 16 * sum(c for j, c in enumerate(send_c) if j != rank)
        n_marks = 7

        def step(evs=None):
            mark(evs, 0)
            ctx.legendre_alm2map_dev(alm.data_ptr(), send.data_ptr())
            mark(evs, 1)
            dist.all_to_all_single(recv, send, r_split, s_split)
            mark(evs, 2)
            ctx.ring_synthesis_dev(recv.data_ptr(), mp.data_ptr())
            mark(evs, 3)
            ctx.ring_analysis_dev(mp.data_ptr(), recv.data_ptr())
            mark(evs, 4)
            dist.all_to_all_single(send, recv, s_split, r_split)
            mark(evs, 5)
            ctx.legendre_map2alm_dev(send.data_ptr(), alm_out.data_ptr())
            mark(evs, 6)

        def stages(evs):
            return (evs[0].elapsed_time(evs[1]), evs[2].elapsed_time(evs[3]), evs[3].elapsed_time(evs[4]),
                    evs[5].elapsed_time(evs[6]), evs[1].elapsed_time(evs[2]) + evs[4].elapsed_time(evs[5]))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if use_exchange:
        import torch.distributed as dist
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_marks)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        if use_exchange:
            dist.barrier()
        ev0.record(stream)
        n_launch0 = sht.kernel_launches()
        for i in range(args.steps):  # no host synchronisation inside the timed region
            step(step_evs[i])
        ev1.record(stream)
        n_launches = sht.kernel_launches() - n_launch0  # the library's own kernels, timed region
        torch.cuda.synchronize(dev)
        if use_exchange:
            dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    if use_exchange:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps

    # ---- stage times of the timed steps (their events, read after the region) ----
    st = np.array([stages(evs) for evs in step_evs])  # steps x (leg a2m, synth, anal, leg m2a, exch)
    leg_s, fft_s, fft_a, leg_a, exch_ms = st[:, 0], st[:, 1], st[:, 2], st[:, 3], list(st[:, 4])

    # ---- end to end through the host-buffer C ABI (pinned host memory) ----
    e2e = None
    if ws == 1:
        alm_pin = torch.from_numpy(alm_h.view(np.float64)).pin_memory()
        map_pin = torch.empty(grid.n_pix, dtype=torch.float64).pin_memory()
        alm_back = torch.empty_like(alm_pin).pin_memory()
        a_np = alm_pin.numpy().view(np.complex128)
        m_np = map_pin.numpy()
        b_np = alm_back.numpy().view(np.complex128)
        for _ in range(max(1, args.warmup // 2)):
            ctx.alm2map(a_np, out=m_np)
            ctx.map2alm(m_np, out=b_np)
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_launch_e0 = sht.kernel_launches()
        for _ in range(args.steps):
            ctx.alm2map(a_np, out=m_np)
            ctx.map2alm(m_np, out=b_np)
        e1.record(stream)
        n_launch_e2e = sht.kernel_launches() - n_launch_e0
        torch.cuda.synchronize(dev)
        e2e_ms = e0.elapsed_time(e1) / args.steps
        bytes_alm = n_alm * 16
        bytes_map = grid.n_pix * 8
        e2e = {"value": 2 * falg_flops(lmax, mmax, grid.n_rings) / (e2e_ms * 1e-3) / 1e12,
               "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": bytes_alm + bytes_map, "d2h_bytes_per_step": bytes_map + bytes_alm,
               "gpu_launches": n_launch_e2e, "host_memory": "page-locked (pinned torch tensors)"}
        # the path a reference C++ user hits: pageable std::vector-like buffers (numpy), which
        # the library stages through its own page-locked buffers (wall clock: the call returns
        # when the output is in place)
        a_pg = alm_h.copy()
        m_pg = np.empty(grid.n_pix)
        b_pg = np.empty_like(alm_h)
        ctx.alm2map(a_pg, out=m_pg)
        ctx.map2alm(m_pg, out=b_pg)
        n_pg = min(args.steps, 5)
        t0 = time.perf_counter()
        for _ in range(n_pg):
            ctx.alm2map(a_pg, out=m_pg)
            ctx.map2alm(m_pg, out=b_pg)
        pg_ms = (time.perf_counter() - t0) * 1e3 / n_pg
        e2e["pageable"] = {"value": 2 * falg_flops(lmax, mmax, grid.n_rings) / (pg_ms * 1e-3) / 1e12,
                           "unit": "TFLOP/s", "ms_per_step": pg_ms, "steps": n_pg,
                           "host_memory": "pageable (numpy), staged by the library on all host cores"}
        # first call on a fresh context: geometry + band + plan (recurrence tables, activation
        # scan, FFT tables) + one alm2map + one map2alm from pinned host buffers (wall clock)
        t0 = time.perf_counter()
        cold = sht.Context(local)
        cold.set_stream(stream.cuda_stream)
        cold.set_grid(grid, mirror=True)
        cold.set_band(lmax, mmax)
        t1 = time.perf_counter()
        cold.plan()
        t2 = time.perf_counter()
        cold.alm2map(a_np, out=m_np)
        cold.map2alm(m_np, out=b_np)
        t3 = time.perf_counter()
        cold.close()
        e2e["first_call"] = {"ms": (t3 - t0) * 1e3, "plan_ms": (t2 - t1) * 1e3,
                             "transforms_ms": (t3 - t2) * 1e3, "setup_ms": (t1 - t0) * 1e3,
                             "note": "fresh context: set_grid + set_band + plan + alm2map + map2alm, "
                                     "pinned host buffers, wall clock"}
    elif args.exchange == "peer":
        # N ranks: every rank reads its orders' a_lm from a pinned host triangle, runs the fused
        # m-distributed step, writes its rings' pixels to a pinned host map, reads them back as
        # the map2alm input and writes its orders' a_lm back; copies on the shared stream
        # (not pipelined against the kernels), max over ranks
        alm_pin = torch.from_numpy(alm_h.view(np.float64)).pin_memory()
        map_pin = torch.zeros(grid.n_pix, dtype=torch.float64).pin_memory()
        alm_back = torch.zeros_like(alm_pin).pin_memory()
        ivs = []  # this rank's rings as pixel intervals
        offs, nphi = np.asarray(grid.pixel_offset), np.asarray(grid.n_phi)
        for r in sorted(layout.ring_sets[rank]):
            b, e = int(offs[r]), int(offs[r] + nphi[r])
            if ivs and ivs[-1][1] == b:
                ivs[-1][1] = e
            else:
                ivs.append([b, e])
        alm_dev = torch.empty_like(alm)

        def e2e_step():
            ctx.copy_orders(alm_pin.data_ptr(), alm_dev.data_ptr(), True)
            ctx.legendre_alm2map_peer(alm_dev.data_ptr())
            px.barrier()
            ctx.ring_synthesis_dev(px.recv, mp.data_ptr())
            for b, e in ivs:
                map_pin[b:e].copy_(mp[b:e], non_blocking=True)
            for b, e in ivs:
                mp[b:e].copy_(map_pin[b:e], non_blocking=True)
            ctx.ring_analysis_peer(mp.data_ptr())
            px.barrier()
            ctx.legendre_map2alm_dev(px.send, alm_out.data_ptr())
            ctx.copy_orders(alm_out.data_ptr(), alm_back.data_ptr(), False)
        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_launch_e0 = sht.kernel_launches()
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        n_launch_e2e = sht.kernel_launches() - n_launch_e0
        torch.cuda.synchronize(dev)
        dist.barrier()
        own_alm = sum(lmax - m + 1 for m in layout.m_sets[rank]) * 16
        own_map = sum(e - b for b, e in ivs) * 8
        t = torch.tensor([e0.elapsed_time(e1), float(own_alm + own_map)], dtype=torch.float64,
                         device="cpu" if shared else dev)
        tm = t.clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e2e_ms = float(tm[0].item()) / args.steps
        moved = int(t[1].item())  # whole job, each direction
        e2e = {"value": 2 * falg_flops(lmax, mmax, grid.n_rings) / (e2e_ms * 1e-3) / 1e12,
               "unit": "TFLOP/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": moved,
               "d2h_bytes_per_step": moved, "gpu_launches": n_launch_e2e,
               "note": "per rank: its orders' a_lm and its rings' pixels over its own PCIe link, "
                       "copies not pipelined against the kernels"}

    # ---- parity spot check of the timed output (the reference is checked in tests/) ----
    roundtrip = None
    if ws == 1:
        back = alm_out.cpu().numpy().view(np.complex128)
        roundtrip = float(np.linalg.norm(back - alm_h) / np.linalg.norm(alm_h))

    if rank != 0:
        if use_exchange:
            dist.destroy_process_group()
        return

    fl_step = 2 * falg_flops(lmax, mmax, grid.n_rings)
    value = fl_step / (ms_step * 1e-3) / 1e12
    peak_tf, _ = sht.measure_fp64_peak(local)
    leg_a_ms, leg_s_ms = float(np.mean(leg_a)), float(np.mean(leg_s))
    fl_leg = falg_flops(lmax, mmax, grid.n_rings) / ws  # per rank, per launch
    dom_ms, dom_name = (leg_a_ms, "leg_map2alm_kernel") if leg_a_ms >= leg_s_ms else (leg_s_ms, "leg_alm2map_kernel")
    # headline basis: the (l, m, ring-pair) steps the kernel actually executes x 8 flops (dead
    # and never-activating streams are skipped, so the F_alg basis would count work that never
    # runs); F_alg = 8 x n_alm x ceil(R_N/2) is kept as the secondary figure
    # this rank's plan, per launch: map2alm runs tile pairs, alm2map single tiles
    exec_a2m = 8.0 * stats.get("executed_alm2map", stats["executed"])
    exec_m2a = 8.0 * stats.get("executed_map2alm", stats["executed"])
    exec_fl = exec_m2a if dom_name == "leg_map2alm_kernel" else exec_a2m
    achieved = exec_fl / (dom_ms * 1e-3) / 1e12
    falg_achieved = fl_leg / (dom_ms * 1e-3) / 1e12
    # DRAM bytes per launch and ncu-executed DP rate from the committed full capture
    traffic, ncu_rec = None, {}
    tf = ROOT / "profiles" / "ncu_kernels.json"
    if tf.exists():
        try:
            ncu_rec = json.loads(tf.read_text()).get(dom_name, {})
            traffic = ncu_rec.get("dram_bytes")
        except Exception:
            traffic, ncu_rec = None, {}
    roofline = {
        "bound": "fp64", "kernel": dom_name, "achieved": achieved, "peak": peak_tf,
        "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic,
        "basis": "executed: 8 flops x (l, m, ring-pair) steps the kernel runs (plan count, "
                 "cross-checked against ncu's executed DP instructions)",
        "peak_source": "measured live: DFMA-loop probe (shtc_measure_fp64_peak); "
                       "MEASURED_PEAKS.json has no FP64 entry",
        "flops_per_launch": exec_fl,
        "falg": {"achieved": falg_achieved, "frac": falg_achieved / peak_tf, "flops_per_launch": fl_leg,
                 "basis": "algorithmic 8 x n_alm x ceil(R_N/2) (reference mirror-path steps x 8; "
                          "counts the skipped dead-stream steps)"},
        "useful_tflops": 8.0 * stats["useful"] / (dom_ms * 1e-3) / 1e12,
        "ncu": {"executed_dp_tflops": ncu_rec.get("executed_dp_tflops"),
                "fp64_pipe_pct": ncu_rec.get("fp64_pipe_pct"), "source": ncu_rec.get("source")},
        "alm2map_kernel": {"ms": leg_s_ms, "achieved": exec_a2m / (leg_s_ms * 1e-3) / 1e12,
                           "falg_achieved": fl_leg / (leg_s_ms * 1e-3) / 1e12},
        "map2alm_kernel": {"ms": leg_a_ms, "achieved": exec_m2a / (leg_a_ms * 1e-3) / 1e12,
                           "falg_achieved": fl_leg / (leg_a_ms * 1e-3) / 1e12},
    }
    ms_a2m = float(np.mean(leg_s)) + float(np.mean(fft_s))
    ms_m2a = float(np.mean(leg_a)) + float(np.mean(fft_a))
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Gaussian a_lm (splitmix64 counter stream + Box-Muller, seed 12345); "
                "map2alm input = the step's alm2map output",
        "config": {"workload": f"alm2map+map2alm HEALPix nside={args.nside} lmax=mmax={lmax}{config_tag(args.nside, lmax)}",
                   "grid": "healpix-ring", "nside": args.nside, "lmax": lmax, "mmax": mmax,
                   "parallelism": f"m-distributed x{ws}" + {"none": "", "peer": " + fused peer-memory exchange",
                                                            "nccl": " + NCCL all-to-all"}[args.exchange],
                   "l2": l2_note(n_alm, grid.n_pix, grid.n_rings, mmax)},
        "ms_alm2map": ms_a2m, "ms_map2alm": ms_m2a,
        "stages_ms": {"alm2map": {"legendre": leg_s_ms, "fft": float(np.mean(fft_s))},
                      "map2alm": {"legendre": leg_a_ms, "fft": float(np.mean(fft_a))}},
        "plan_s": plan_s, "steps_accounting": stats,
        "exchange": ({"impl": ("Delta stored straight into the owners' buffers by the Legendre / ring-analysis "
                              "kernels (CUDA IPC peer memory over NVLink) + device-side barrier; "
                              "ms_per_step = the two barrier waits" if args.exchange == "peer" else
                              "NCCL all_to_all_single on packed Delta (no pack/unpack kernels)"),
                      "bytes_sent_per_rank_per_transform": exch_bytes,
                      "ms_per_step": float(np.mean(exch_ms[-args.steps:])),
                      "GBps_per_rank": 2 * exch_bytes / (float(np.mean(exch_ms[-args.steps:])) * 1e-3) / 1e9
                      if np.mean(exch_ms[-args.steps:]) > 0 else None}
                     if use_exchange else None),
        "roundtrip_rel_err": roundtrip,
        "clocks": clk.summary(), "e2e": e2e, "roofline": roofline,
        "gpu_launches": n_launches,
    }
    if ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.nside, lmax)
        except Exception as exc:  # the oracle must exist; report instead of hiding
            line["cpu_baseline"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    if use_exchange:
        dist.destroy_process_group()


def run_reference(args):
    """The reference arm: the reference's CPU implementation (oracle/_ref) on all host threads,
    every step = one alm2map + one map2alm at the workload's own config (C4 by default, ~13 s
    on 16 cores).  Warm-up on a CPU only touches the caches and thread pool, so at most one
    warm-up step runs (keeps `--steps 20 --warmup 5` at ~4.5 minutes)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    for _ in range(min(args.warmup, 1)):
        cpu_baseline(args.nside, args.lmax)
    steps = [cpu_baseline(args.nside, args.lmax) for _ in range(args.steps)]
    ms_step = float(np.median([s["ms_per_step"] for s in steps]))
    v = 2 * falg_flops(args.lmax, args.lmax, 4 * args.nside - 1) / (ms_step * 1e-3) / 1e12
    cb = dict(steps[-1])
    cb["value"] = v
    cb["ms_per_step"] = ms_step
    cb["sample"] = cb["sample"] + f"; median of {args.steps} steps"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "warmup_run": min(args.warmup, 1),
        "ms_per_step": ms_step,
        "ms_alm2map": float(np.median([s["ms_alm2map"] for s in steps])),
        "ms_map2alm": float(np.median([s["ms_map2alm"] for s in steps])),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Gaussian a_lm (splitmix64 counter stream + Box-Muller, seed 12345); "
                "map2alm input = the step's alm2map output",
        "config": {"workload": f"alm2map+map2alm HEALPix nside={args.nside} lmax=mmax={args.lmax}"
                               f"{config_tag(args.nside, args.lmax)}",
                   "grid": "healpix-ring", "nside": args.nside, "lmax": args.lmax, "mmax": args.lmax,
                   "parallelism": f"reference CPU, 1 worker x {cb['cores']} threads",
                   "sample": cb["sample"]},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def ensure_world(args):
    """`python bench.py --gpus N` runs N ranks: outside torchrun (no WORLD_SIZE) with N > 1 the
    script re-executes itself under torch.distributed.run, one process per GPU; inside torchrun
    the world size must equal N."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
            sys.stdout.flush()
            os.execv(sys.executable, cmd)
        return
    if int(ws) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--nside", type=int, default=NSIDE)
    p.add_argument("--lmax", type=int, default=LMAX)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--exchange", choices=["auto", "none", "peer", "nccl"], default="auto",
                   help="Delta exchange of the m-distributed path: peer (fused stores over peer "
                        "memory, the default for N>1), nccl (packed all_to_all_single), none (N=1 "
                        "whole transforms, the default for N=1); peer/nccl also run at N=1")
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    ensure_world(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
