"""CPU: the C-ABI libraries load and export every symbol include/*.h declares; with no CUDA
device the product fails loudly (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared(header: Path):
    txt = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(shtc_[a-z0-9_]+)\s*\(", txt)))


def test_libshtc_exports_every_declared_symbol():
    from paper_1106_0159_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared(ROOT / "include" / "shtc.h")
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTED)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_1106_0159_b200 import sht
    with pytest.raises(Exception) as ei:
        sht.Context(0)
    assert str(ei.value)


def test_reference_oracle_library_loads():
    from oracle import ref
    assert ref.available()
    assert ref.splitmix64_at(0, 0) == 0xE220A8397B1DCDAF
