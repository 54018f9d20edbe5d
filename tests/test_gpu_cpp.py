"""GPU: the C++ drop-in API (include/sht/*.hpp over libshtc) against the reference, through a
compiled parity program (tests/cpp/dropin_parity.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1106_0159_b200"


@pytest.mark.gpu
def test_cpp_dropin_parity(tmp_path):
    exe = tmp_path / "dropin_parity"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "dropin_parity.cpp"), "-o", str(exe),
                    f"-L{PKG}", "-lsht_b200", "-lshtc", str(ROOT / "oracle" / "_ref" / "libsht_ref.so"),
                    f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ROOT / 'oracle' / '_ref'}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
