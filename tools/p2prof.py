"""Phase timing of the power-of-two ring-synthesis engine (tuning build with -DP2_PROF):

    python -c "from paper_1106_0159_b200 import build as b; b.build_variant('prof', ['P2_PROF'])"
    SHTC_VARIANT_LIB=paper_1106_0159_b200/_build/var_prof/libshtc.so python tools/p2prof.py

Prints thread 0's average cycles per ring for each phase of each class (rings per CTA run
back to back; phases end at the marks P2T(i) in ring_p2_synth_kernel)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1106_0159_b200 import _lib, sht

PH = ["phase-tab", "fold", "fold-sync", "Z-prologue", "sync", "fft1", "H-mult", "fft2", "chirp-out",
      "stores", "end-sync"]
nside, lmax = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 4096)))
g = sht.build_healpix_grid(nside)
ctx = sht.Context(0)
ctx.set_grid(g)
ctx.set_band(lmax, lmax)
ctx.plan()
alm = torch.from_numpy(sht.gaussian_alm(lmax, lmax, 1).view(np.float64)).cuda()
mp = torch.empty(g.n_pix, dtype=torch.float64, device="cuda")
delta = torch.empty(2 * g.n_rings * (lmax + 1), dtype=torch.float64, device="cuda")
L = _lib.lib()
buf = (C.c_ulonglong * 256)()
ctx.legendre_alm2map_dev(alm.data_ptr(), delta.data_ptr())
ctx.ring_synthesis_dev(delta.data_ptr(), mp.data_ptr(), timing=True)
L.shtc_p2prof(buf, 1)
reps = 5
t = [ctx.ring_synthesis_dev(delta.data_ptr(), mp.data_ptr(), timing=True)["fft_ms"] for _ in range(reps)]
torch.cuda.synchronize()
L.shtc_p2prof(buf, 0)
a = np.frombuffer(buf, dtype=np.uint64).reshape(16, 16).astype(np.float64)
print(f"ring synthesis {np.median(t):.3f} ms")
for slot in range(16):
    rings = a[slot, 15]
    if rings == 0:
        continue
    M = 1 << (slot % 8 + 8)
    kind = "bluestein" if slot >= 8 else "direct"
    row = a[slot, :11] / rings
    print(f"M={M:5d} {kind:9s} rings/rep={rings / reps:7.0f} total={row.sum():8.0f} cyc/ring | " +
          " ".join(f"{PH[i]}={row[i]:.0f}" for i in range(11) if row[i] > 0))
