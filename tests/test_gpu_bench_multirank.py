"""The N > 1 bench path end to end (torchrun, one process per rank, m-distributed plan, fused
peer-memory exchange, device-side barrier, max-over-ranks timing, one JSON line from rank 0),
run on the one GPU this environment has: SHT_BENCH_SHARED_GPU=1 puts every rank on device 0
and uses gloo for the control plane.  The per-rank results are checked bitwise against one
worker in tests/test_gpu_peer_exchange.py; this test covers the driver's launch sequence."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [2, 3])
def test_bench_multirank_shared_gpu(n):
    # exactly the driver's form `python bench.py --gpus N` (no torchrun wrapper): bench.py
    # re-executes itself under torch.distributed.run with N ranks
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["SHT_BENCH_SHARED_GPU"] = "1"
    cmd = [sys.executable, "bench.py", "--gpus", str(n),
           "--steps", "3", "--warmup", "3", "--nside", "128", "--lmax", "256"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["steps"] == 3 and d["ms_per_step"] > 0
    assert "peer-memory exchange" in d["config"]["parallelism"]
    assert d["exchange"]["bytes_sent_per_rank_per_transform"] > 0
    assert d["gpu_launches"] > 0
    # end to end through pinned host buffers at N ranks: the whole job's a_lm + map each way
    assert d["e2e"]["ms_per_step"] > 0 and d["e2e"]["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 16 * (257 * 258 // 2) + 8 * 12 * 128 * 128

