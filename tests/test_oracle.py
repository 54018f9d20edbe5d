"""CPU: the oracle restatement (oracle/sht_oracle.py) pinned against the reference's golden
vectors (tests/golden/*.npz, made by tests/golden/make_golden.py from oracle/_ref) and the
known-answer constants of the reference unit tests (test_legendre.cpp, test_experiment.cpp)."""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import sht_oracle as O

G = Path(__file__).resolve().parent / "golden"


class Grid:
    def __init__(self, d):
        self.cos_theta, self.n_phi, self.phi_0, self.weight = d["cos_theta"], d["n_phi"], d["phi_0"], d["weight"]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_mu_beta_plm_kats():
    # test_legendre.cpp:46-54, 56-64, 83-87
    assert math.exp(O.log_mu(0)) == pytest.approx(0.28209479177387814, rel=1e-13)
    assert math.exp(O.log_mu(1)) == pytest.approx(0.34549414947133548, rel=1e-13)
    assert math.exp(O.log_mu(2)) == pytest.approx(0.38627420202318958, rel=1e-13)
    assert O.beta_lm(2, 0) == pytest.approx(1.9364916731037084, rel=1e-14)
    assert O.beta_lm(3, 1) == pytest.approx(2.0916500663351889, rel=1e-14)
    assert O.plm_row(0, 0.5, 1)[1] == pytest.approx(0.24430125595145996, rel=1e-13)
    assert O.plm_row(1, 0.5, 1)[0] == pytest.approx(0.29920671030107451, rel=1e-13)
    with pytest.raises(ArithmeticError):
        O.beta_lm(1, 1)
    with pytest.raises(ValueError):
        O.beta_lm(1, 2)


def test_kats_match_reference_golden():
    k = np.load(G / "kat.npz")
    for m, v in zip(k["log_mu_m"], k["log_mu"]):
        assert O.log_mu(int(m)) == pytest.approx(float(v), rel=1e-13, abs=1e-12)
    assert O.beta_lm(2, 0) == float(k["beta_20"])
    assert O.beta_lm(3, 1) == float(k["beta_31"])
    assert O.plm_row(0, 0.5, 1)[1] == pytest.approx(float(k["plm_10_05"]), rel=1e-15)
    assert [O.splitmix64_at(0, i) for i in range(3)] == [int(v) for v in k["splitmix_0"]]
    # test_experiment.cpp:49-51
    assert O.splitmix64_at(0, 0) == 0xE220A8397B1DCDAF
    assert O.splitmix64_at(0, 1) == 0x6E789E6AA1B965F4
    assert O.splitmix64_at(0, 2) == 0x06C45D188009454F
    assert sum(O.assign_m(7, 2), []) == list(k["assign_m_7_2"])
    assert sum(O.assign_m(7, 4), []) == list(k["assign_m_7_4"])
    assert sum(O.assign_rings(7, 2), []) == list(k["assign_rings_hp2_2"])
    assert np.allclose(O.ring_synthesis(np.array([0, 1], complex), 4, 0.0), k["ring_synth_4"], atol=1e-14)


def test_deep_order_scaled_row():
    """m=2000, lmax=2200, x=0.999 (test_legendre.cpp:167-224): ladder scales and mantissas."""
    k = np.load(G / "kat.npz")
    mant, sc = O.plm_row_scaled(2000, 0.999, 2200)
    assert np.array_equal(sc, k["deep_scale"])
    assert sc[0] < -10
    assert np.max(np.abs(mant - k["deep_mant"]) / np.abs(k["deep_mant"])) < 1e-12


@pytest.mark.parametrize("name", ["hp4_l12", "hp8_l20", "gl17_l16", "gl10_l9", "gl9_nphi7_l8"])
def test_transforms_match_reference_golden(name):
    d = np.load(G / f"transform_{name}.npz")
    lmax = int(d["lmax"])
    g = Grid(d)
    alm = O.random_alm(lmax, lmax, int(d["seed"]))
    assert np.array_equal(alm, d["alm"])
    mp = O.synthesis(alm, lmax, lmax, g)
    assert rel(mp, d["map"]) < 1e-13
    back = O.analysis(d["map"], lmax, lmax, g)
    assert rel(back, d["alm_back"]) < 1e-13
    # the reference's step counters (transforms.cpp:178): nominal = pairs * sum(lmax-m+1)
    per = sum(lmax - m + 1 for m in range(lmax + 1))
    assert int(d["steps_paired"]) == ((len(g.cos_theta) + 1) // 2) * per
    assert int(d["steps_unpaired"]) == len(g.cos_theta) * per


def test_legendre_operators_match_reference_golden():
    d = np.load(G / "operators_gl17.npz")
    panel = O.compute_delta_a(d["alm"], 16, 16, d["x"], list(d["ms"]))
    # same operation order as the reference: bit for bit
    assert np.array_equal(panel, d["panel"])
