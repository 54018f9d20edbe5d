"""Generate the golden fixtures from the reference itself (oracle/_ref, compiled from
/root/reference/proj/src by oracle/build_ref.sh).  Run in the authoring container:

    python tests/golden/make_golden.py

The fixtures are small .npz files committed next to this script; the CPU suite checks the
oracle restatement and the host-side code against them, the GPU suite checks the CUDA path.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent


def grid_arrays(g):
    return dict(cos_theta=g.cos_theta, n_phi=g.n_phi, phi_0=g.phi_0, weight=g.weight,
                pixel_offset=g.pixel_offset)


def main():
    # ---- known-answer values of the reference unit tests -------------------------------
    kat = {
        "log_mu": np.array([ref.log_mu(m) for m in range(0, 12)] + [ref.log_mu(2000), ref.log_mu(4096)]),
        "log_mu_m": np.array(list(range(0, 12)) + [2000, 4096]),
        "beta_20": ref.beta_lm(2, 0), "beta_31": ref.beta_lm(3, 1),
        "plm_10_05": ref.plm_row(0, 0.5, 1)[1], "plm_11_05": ref.plm_row(1, 0.5, 1)[0],
        "splitmix_0": np.array([ref.splitmix64_at(0, i) for i in range(3)], dtype=np.uint64),
        "assign_m_7_2": np.array(sum(ref.assign_m(7, 2), [])),
        "assign_m_7_4": np.array(sum(ref.assign_m(7, 4), [])),
        "assign_rings_hp2_2": np.array(sum(ref.assign_rings_healpix(2, 2), [])),
        "ring_synth_4": ref.ring_synthesis(np.array([0, 1], np.complex128), 4, 0.0),
    }
    m, sc = ref.plm_row_scaled(2000, 0.999, 2200)
    kat["deep_mant"], kat["deep_scale"] = m, sc
    for k in range(1, 4):
        kat[f"hp{k}"] = np.stack([ref.healpix_grid(k).cos_theta, ref.healpix_grid(k).n_phi.astype(float),
                                  ref.healpix_grid(k).phi_0])
    np.savez_compressed(OUT / "kat.npz", **kat)

    # ---- transforms -----------------------------------------------------------------------
    cases = {}
    for name, g, lmax, seed in [("hp4_l12", ref.healpix_grid(4), 12, 12345),
                                ("hp8_l20", ref.healpix_grid(8), 20, 77),
                                ("gl17_l16", ref.gl_grid(17, 34), 16, 555),
                                ("gl10_l9", ref.gl_grid(10, 24), 9, 91),
                                ("gl9_nphi7_l8", ref.gl_grid(9, 7), 8, 3)]:
        alm = ref.random_alm(lmax, lmax, seed)
        mp, steps = ref.synthesis(alm, lmax, lmax, g, pairing=True)
        mp_u, steps_u = ref.synthesis(alm, lmax, lmax, g, pairing=False)
        back, _ = ref.analysis(mp, lmax, lmax, g, pairing=True)
        d = dict(lmax=lmax, seed=seed, alm=alm, map=mp, map_unpaired=mp_u, alm_back=back,
                 steps_paired=steps, steps_unpaired=steps_u, **grid_arrays(g))
        np.savez_compressed(OUT / f"transform_{name}.npz", **d)
        cases[name] = mp.size
    # ---- Legendre operators (test_transforms.cpp:99-148) ----------------------------------
    x, _ = ref.gl_nodes(17)
    alm = ref.random_alm(16, 16, 555)
    ms = np.arange(17)
    panel, steps = ref.compute_delta_a(alm, 16, 16, x, ms)
    rng = np.random.default_rng(808)
    dpanel = rng.uniform(-1, 1, (17, 17)) + 1j * rng.uniform(-1, 1, (17, 17))
    acc, _ = ref.accumulate_alm(dpanel, x, ms, 16, 16)
    np.savez_compressed(OUT / "operators_gl17.npz", x=x, alm=alm, ms=ms, panel=panel, steps=steps,
                        dpanel=dpanel, acc=acc)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
