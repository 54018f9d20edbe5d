"""file containers, CLI edge and the recalibrated performance model.
CPU parts run here; the CLI transforms run on the GPU and are checked against the reference."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1106_0159_b200"
CLI = PKG / "sht_b200"


def _build(tmp, src, name):
    exe = tmp / name
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    f"-L{PKG}", "-lsht_b200", "-lshtc", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def test_edge_cpu_program(tmp_path):
    exe = _build(tmp_path, ROOT / "tests" / "cpp" / "edge_cpu.cpp", "edge_cpu")
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def run_cli(*args, check=True):
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


def test_cli_grid_partition_model():
    out = run_cli("grid", "info", "--nside", 4).stdout
    assert "rings 15" in out and "pixels 192" in out
    out = run_cli("partition", "--grid", "gauss-legendre", "--nrings", 8, "--nphi", 16, "--lmax", 7,
                  "--workers", 2, "--threads", 2).stdout
    assert "worker 0 m { 0 2 5 7 }" in out and "worker 1 rings { 2 3 4 5 }" in out
    assert "worker 0 thread 0 m { 0 7 }" in out
    csv = run_cli("model", "--nside", 64, "--workers", 1, "--workers", 4).stdout.strip().splitlines()
    assert csv[0] == "nside,lmax,mmax,n_workers,precompute_s,compute_s,comm_s,ratio"
    f = [float(x) for x in csv[2].split(",")]
    # compute_s = gamma * (c2 r l m / n + c3 (r/n) m log2 m) with the reference constants
    r, l = 255.0, 128.0
    want = 1e-10 * (4 * r * l * l / 4 + 5 * (r / 4) * l * np.log2(l))
    assert abs(f[5] - want) <= 1e-12 * want
    assert run_cli("synth", "--bogus", check=False).returncode == 1


def read_shtmap(path):
    raw = Path(path).read_bytes()
    head, body = raw.split(b"end\n", 1)
    return head.decode(), np.frombuffer(body, "<f8")


@pytest.mark.gpu
def test_cli_synth_analyze_match_reference(tmp_path):
    from oracle import ref
    nside, lmax = 16, 32
    run_cli("synth", "--nside", nside, "--lmax", lmax, "--seed", 99, "--out", tmp_path / "m.shtmap")
    head, mp = read_shtmap(tmp_path / "m.shtmap")
    assert head.startswith("SHTMAP1\nscheme healpix-ring\nnside 16\n")
    g = ref.healpix_grid(nside)
    want, _ = ref.synthesis(ref.random_alm(lmax, lmax, 99), lmax, lmax, g, pairing=True)
    assert np.linalg.norm(mp - want) / np.linalg.norm(want) < 1e-12
    run_cli("analyze", tmp_path / "m.shtmap", "--lmax", lmax, "--out", tmp_path / "a.shtalm")
    head, a = read_shtmap(tmp_path / "a.shtalm")
    assert head.startswith("SHTALM1\nlmax 32\nmmax 32\n")
    wa, _ = ref.analysis(want, lmax, lmax, g, pairing=True)
    a = a.view(np.complex128)
    assert np.linalg.norm(a - wa) / np.linalg.norm(wa) < 1e-12
    out = run_cli("roundtrip", "--nside", nside, "--lmax", lmax, "--workers", 2).stdout
    assert "D_err" in out
    out = run_cli("bench", "--nside", nside, "--lmax", lmax, "--workers", 2, "--threads", 2).stdout
    assert out.startswith("stage,predicted_s,measured_s,flops,bytes")
    assert "recurrence_steps" in out
