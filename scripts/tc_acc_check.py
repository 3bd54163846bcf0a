import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.subspace import gram_matrix
from paper_2004_08962_b200.synthetic import make_config
from oracle import hicu_oracle as O
dims, kext = (256, 256, 8), (5, 5, 8)
rng = np.random.default_rng(0)
for kind in ("random", "phantom"):
    if kind == "random":
        x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64)
    else:
        k16, m16, x016 = make_config("C2")
        xc, _, _ = O.coil_compress(k16, m16, 8)
        x = xc.astype(np.complex64)
    k = H.KernelMask.full(kext)
    reg = H.full_region(dims, k)
    Gr = O.gram(x.astype(np.complex128), O.full_geom(dims, kext))
    for force in (False, True):
        G = gram_matrix(x, k, reg, force_simt=force).cpu().numpy()
        E = np.abs(G - Gr)
        d = np.diag(E).max() / np.abs(np.diag(Gr)).max()
        off = (E - np.diag(np.diag(E))).max() / np.abs(Gr).max()
        rel_each = (E / np.maximum(np.abs(Gr), 1e-30 * np.abs(Gr).max())).max()
        print(kind, "simt" if force else "tc  ", os.environ.get("HICU_TC_MAX_KB", "-"), f"diag {d:.2e} off/max {off:.2e} maxrel/max {E.max() / np.abs(Gr).max():.2e}", flush=True)
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry
dg = device_geometry(H.KernelMask.full(kext), H.full_region(dims, H.KernelMask.full(kext)), dims)
print("workspace bytes", nat.lib().hicu_gram_workspace(dg.ref()), "env", os.environ.get("HICU_TC_MAX_KB"))
