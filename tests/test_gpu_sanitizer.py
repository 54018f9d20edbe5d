"""Race and memory checking of the CUDA path (compute-sanitizer on a small case).

tools/sanitize_run.py drives every kernel family through the C ABI (pipelined host paths,
ring classes, Legendre operators) and checks the results against the reference; here it runs
under compute-sanitizer's memcheck (out-of-bounds / misaligned accesses), racecheck
(shared-memory hazards) and synccheck (barrier misuse), each of which must report no error.
"""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _sanitizer():
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and Path(cand).exists():
            return cand
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "3", "--print-limit", "20",
           sys.executable, str(ROOT / "tools" / "sanitize_run.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:
        # the GPU pool refuses sanitizer runs; the same workload still runs (every kernel
        # family against the reference), the sanitizer verdict stays the one recorded in
        # profiles/r01_sanitizer.txt
        w = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_run.py")], cwd=ROOT,
                           capture_output=True, text=True, timeout=1200)
        assert w.returncode == 0 and "sanitize_run ok" in w.stdout + w.stderr, (w.stdout + w.stderr)[-4000:]
        pytest.skip("compute-sanitizer closed on this GPU pool (workload checked without it)")
    assert r.returncode == 0, out[-4000:]
    assert "sanitize_run ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
