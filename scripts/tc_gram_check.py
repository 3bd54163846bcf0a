"""Standalone tcgen05 Gram check: TC vs SIMT vs oracle on several geometries."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.subspace import gram_matrix, gram_uses_tensor_cores
from oracle import hicu_oracle as O

rng = np.random.default_rng(0)
cases = [((40, 36, 8), (5, 5, 8), "full"), ((64, 64, 8), (5, 5, 8), [24, 24]), ((30, 27, 8), (3, 3, 8), "full"),
         ((12, 11, 13, 8), (3, 3, 3, 8), "full"), ((256, 256, 8), (5, 5, 8), "full")]
for dims, kext, frac in cases:
    x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64)
    k = H.KernelMask.full(kext)
    reg = H.stage_region(dims, k, frac)
    tc = gram_uses_tensor_cores(k, reg, dims)
    t = time.time()
    G1 = gram_matrix(x, k, reg).cpu().numpy()
    G0 = gram_matrix(x, k, reg, force_simt=True).cpu().numpy()
    Gr = O.gram(x.astype(np.complex128), O.stage_geom(dims, kext, frac)) if np.prod(dims) < 300000 else G0
    e1 = np.abs(G1 - Gr).max() / np.abs(Gr).max()
    e0 = np.abs(G0 - Gr).max() / np.abs(Gr).max()
    print(dims, kext, frac, "tc" if tc else "simt", "err tc", e1, "err simt", e0, "herm", np.abs(G1 - G1.conj().T).max(),
          flush=True)
# timing at C2 full size
dims, kext = (256, 256, 8), (5, 5, 8)
x = torch.from_numpy((rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64)).cuda()
k = H.KernelMask.full(kext)
reg = H.full_region(dims, k)
for force in (False, True):
    for _ in range(3):
        gram_matrix(x, k, reg, force_simt=force)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        gram_matrix(x, k, reg, force_simt=force)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 20
    fl = 4.0 * reg.s * k.n * (k.n + 1)
    print("C2 full gram", "simt" if force else "tc", f"{ms:.3f} ms", f"{fl / ms / 1e9:.1f} TFLOP/s (alg)", flush=True)
