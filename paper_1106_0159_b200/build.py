"""Build recipe for the in-tree native libraries (nvcc, sm_100a only).

    python -m paper_1106_0159_b200.build            # libshtc.so (+ libsht_b200.so drop-in)

Outputs land next to this file so `gpurun` ships them to the GPU box (they are git-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libshtc.so"
DROPIN_LIB = PKG / "libsht_b200.so"
CLI_BIN = PKG / "sht_b200"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-O2", "-Xptxas", "-v"] + ARCH
CU_SOURCES = ["legendre.cu", "ringfft.cu", "shtc.cu", "group.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if log is not None:
        log.write(r.stderr)
    return r


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "shtc.h"]
    hdr_mtime = max(h.stat().st_mtime for h in headers)
    objs, jobs = [], []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_mtime):
            jobs.append([nvcc(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)])
    ptxas_log = OBJ / "ptxas.log"
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(_run, jobs))
        with open(ptxas_log, "w") as f:
            for r in results:
                f.write(r.stderr)
        if verbose:
            print(ptxas_log.read_text())
    if force or jobs or not LIB.exists():
        _run([nvcc(), "-shared", *ARCH, "-o", str(LIB) + ".tmp", *map(str, objs), "-lcudart", "-ldl"])
        os.replace(str(LIB) + ".tmp", LIB)
    build_dropin(force=force)
    return LIB


def build_dropin(force: bool = False) -> Path:
    """C++ drop-in `sht::` API (include/sht/*.hpp) over the C ABI: libsht_b200.so."""
    srcs = [CSRC / "sht_dropin.cpp", CSRC / "sht_edge.cpp"]
    if not srcs[0].exists():
        return DROPIN_LIB
    hdrs = list((ROOT / "include" / "sht").glob("*.hpp")) + [ROOT / "include" / "shtc.h", CSRC / "hostcopy.h"]
    newest = max(p.stat().st_mtime for p in srcs + hdrs + [LIB, CSRC / "sht_cli.cpp"])
    if not force and DROPIN_LIB.exists() and CLI_BIN.exists() and DROPIN_LIB.stat().st_mtime >= newest:
        return DROPIN_LIB
    _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", str(ROOT / "include"), *map(str, srcs),
          "-o", str(DROPIN_LIB) + ".tmp", f"-L{PKG}", "-lshtc", "-Wl,-rpath,$ORIGIN"])
    os.replace(str(DROPIN_LIB) + ".tmp", DROPIN_LIB)
    # CLI edge (reference tools/sht_main.cpp subcommands) on the drop-in
    _run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(CSRC / "sht_cli.cpp"), "-o",
          str(CLI_BIN) + ".tmp", f"-L{PKG}", "-lsht_b200", "-lshtc", "-Wl,-rpath,$ORIGIN"])
    os.replace(str(CLI_BIN) + ".tmp", CLI_BIN)
    return DROPIN_LIB


def build_variant(name: str, defines: list[str], flags: list[str] | None = None) -> Path:
    """Tuning experiments: libshtc.so rebuilt with extra -D flags into _build/var_<name>/
    (selected at run time with SHTC_VARIANT_LIB; never the shipped library)."""
    d = OBJ / f"var_{name}"
    d.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in CU_SOURCES:
        o = d / (src + ".o")
        objs.append(o)
        jobs.append([nvcc(), *NVCC_FLAGS, *(flags or []), *[f"-D{x}" for x in defines], "-I", str(ROOT / "include"), "-c",
                     str(CSRC / src), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        res = list(ex.map(_run, jobs))
    (d / "ptxas.log").write_text("".join(r.stderr for r in res))
    lib = d / "libshtc.so"
    _run([nvcc(), "-shared", *ARCH, "-o", str(lib), *map(str, objs), "-lcudart", "-ldl"])
    return lib


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "variant":
        print(build_variant(sys.argv[2], sys.argv[3:]))
        sys.exit(0)
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
