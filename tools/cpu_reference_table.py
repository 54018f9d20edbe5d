"""The reference CPU implementation (oracle/_ref: the unmodified sources, Release flags) timed
on this host at C1 and C2, in the variants SURVEY §8(d) asks to report beside the GPU:
all cores with mirror pairing (its fastest path), 1 thread with mirror pairing, and 1 thread
unpaired (the CLI default).  Writes one JSON object.

    python tools/cpu_reference_table.py > profiles/r01_cpu_reference.json
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, ".")
from oracle import ref

F_ALG = lambda lmax, n_rings: 8 * ref.alm_count(lmax, lmax) * ((n_rings + 1) // 2)  # noqa: E731
cores = os.cpu_count() or 1
out = {"host": platform.processor() or platform.machine(), "cores": cores, "configs": {}}
for name, nside, lmax in (("C1", 128, 256), ("C2", 1024, 2048)):
    g = ref.healpix_grid(nside)
    alm = ref.random_alm(lmax, lmax, 12345)
    fl = F_ALG(lmax, len(g.cos_theta))
    row = {}
    for label, fn in (
        (f"{cores} threads, mirror", lambda a, mp=None: ref.distributed_synthesis(a, lmax, lmax, g, n_workers=1,
                                                                                  n_threads=cores, pairing=True)),
        ("1 thread, mirror", lambda a, mp=None: ref.synthesis(a, lmax, lmax, g, pairing=True)),
        ("1 thread, unpaired (CLI default)", lambda a, mp=None: ref.synthesis(a, lmax, lmax, g, pairing=False)),
    ):
        t0 = time.perf_counter()
        mp, _ = fn(alm)
        ts = time.perf_counter() - t0
        if "mirror" in label and label.startswith(str(cores)):
            t0 = time.perf_counter()
            ref.distributed_analysis(mp, lmax, lmax, g, n_workers=1, n_threads=cores, pairing=True)
            ta = time.perf_counter() - t0
        else:
            t0 = time.perf_counter()
            ref.analysis(mp, lmax, lmax, g, pairing="unpaired" not in label)
            ta = time.perf_counter() - t0
        row[label] = {"alm2map_s": round(ts, 4), "map2alm_s": round(ta, 4),
                      "alm2map_GFLOPs_falg": round(fl / ts / 1e9, 2)}
        print(name, label, row[label], file=sys.stderr, flush=True)
    out["configs"][name] = {"nside": nside, "lmax": lmax, "timings": row}
print(json.dumps(out))
