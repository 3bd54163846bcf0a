"""Time the per-iteration nullspace pipeline (Nystrom + Householder +
reflector apply for G=5 JL steps) on a C2 full-stage Gram, p = 8, r = 60.

Usage: python scripts/nullspace_bench.py [reps]   -> one JSON line
Under ncu (warm, --cache-control none) the launch list gives per-kernel times.
"""
import json
import os
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200 import synthetic
from paper_2004_08962_b200.hankel import device_geometry


def main(reps=30):
    ksp, mask, x0 = synthetic.make_config("C2")
    x = x0[..., :8]  # 8 coils (coil compression not needed for timing)
    kernel = H.KernelMask.full((5, 5, 8))
    region = H.full_region(x.shape, kernel)
    G = H.gram_matrix(x.astype(np.complex64), kernel, region)
    n, r, p, gs = kernel.n, 60, 8, 5
    ell = math.ceil(1.5 * r)
    L = nat.lib()
    st = nat.stream_handle()
    rng = np.random.default_rng(0)
    om = torch.from_numpy((rng.standard_normal((n, ell)) + 1j * rng.standard_normal((n, ell))) / np.sqrt(2)).cuda()
    ws_bytes = L.hicu_nystrom_workspace(n, ell)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    V = torch.empty((n, r), dtype=torch.complex128, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    refl = torch.empty(2 * n * r, dtype=torch.complex128, device="cuda")
    tau = torch.empty(r, dtype=torch.complex128, device="cuda")
    flags = torch.zeros(r + 1, dtype=torch.int32, device="cuda")
    jl = not os.environ.get("HICU_NSJL_OFF")
    pbig = torch.zeros((n, gs * p), dtype=torch.complex128, device="cuda")
    pbig[r:] = torch.randn((n - r, gs * p), dtype=torch.complex128, device="cuda")
    B = torch.empty_like(pbig)
    q32 = torch.empty((gs, n, p), dtype=torch.complex64, device="cuda")

    def one():
        nat.check(L.hicu_nystrom(n, ell, r, G.data_ptr(), om.data_ptr(), V.data_ptr(), ws.data_ptr(), ws_bytes,
                                 status.data_ptr(), st), "nystrom")
        if jl:
            nat.check(L.hicu_nullspace_jl(n, r, V.data_ptr(), gs * p, pbig.data_ptr(), B.data_ptr(), q32.data_ptr(), p,
                                          flags[r:].data_ptr(), st), "nullspace_jl")
            return
        nat.check(L.hicu_householder(n, r, V.data_ptr(), 1e-12, refl.data_ptr(), tau.data_ptr(), flags.data_ptr(),
                                     status.data_ptr(), st), "householder")
        nat.check(L.hicu_apply_reflectors(n, r, refl.data_ptr(), tau.data_ptr(), flags.data_ptr(), gs * p,
                                          pbig.data_ptr(), B.data_ptr(), q32.data_ptr(), p, st), "apply")

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        one()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"us_per_iteration": round(e0.elapsed_time(e1) * 1000 / reps, 1), "status": int(status.item()),
                      "n": n, "ell": ell, "r": r}))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 30)
