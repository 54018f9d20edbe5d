"""bench.py's launch contract on CPU: `--gpus N` outside torchrun re-executes under
torch.distributed.run with N ranks (one JSON line from rank 0), a WORLD_SIZE that disagrees
with --gpus is an error, and the reference arm runs the requested config itself (no
projected stand-in config)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(kw)
    return env


def test_world_size_mismatch_fails():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3"], cwd=ROOT,
                       env=_env(WORLD_SIZE="3", RANK="0", LOCAL_RANK="0"),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=3" in (r.stdout + r.stderr)


def test_reference_arm_reexecs_n_ranks_and_keeps_config():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--nside", "16",
                        "--lmax", "32", "--steps", "2", "--warmup", "3"], cwd=ROOT, env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["config"]["nside"] == 16 and d["config"]["lmax"] == 32
    assert "nside=16, lmax=mmax=32" in d["cpu_baseline"]["sample"]
    assert d["ms_alm2map"] > 0 and d["ms_map2alm"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0
