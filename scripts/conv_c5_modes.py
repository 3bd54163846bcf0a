"""Time the three tensor-core convolution calls at the C5 geometry
(256x160x160, 8 coils, 5x5x5x8 kernel, p = 8) under one HICU_CONV_TC_DEBUG
setting (set in the environment: 1 no MMA, 8 no TMEM drain, 2 no TMA):
which role paces the kernel.  Prints one JSON line (us per call)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from conv_tc_bench import run  # noqa: E402

dims = tuple(int(v) for v in os.environ.get("DIMS", "256,160,160,8").split(","))
kext = tuple(int(v) for v in os.environ.get("KEXT", "5,5,5,8").split(","))
t, s, n = run(dims, kext, reps=int(os.environ.get("REPS", "20")), graph_capture=False)
flops = 8 * s * n * 8
print(json.dumps({"debug": os.environ.get("HICU_CONV_TC_DEBUG", "0"), "dims": dims, "us": t,
                  "conv_tflops": round(flops / t["conv_fwd"] / 1e6, 1)}))

if int(os.environ.get("HICU_CONV_TC_DEBUG", "0")) & 32:
    # per-role cycle counters (conv forward): 12 int64 per CTA written into u
    import numpy as np
    import torch
    import paper_2004_08962_b200 as H
    from paper_2004_08962_b200 import _native as nat
    from paper_2004_08962_b200.hankel import device_geometry
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    dg = device_geometry(kernel, region, dims)
    L = nat.lib()
    y = torch.randn(dims, dtype=torch.complex64, device="cuda")
    q = torch.randn((kernel.n, 8), dtype=torch.complex64, device="cuda") / kernel.n ** 0.5
    u = torch.zeros((dg.s, 8), dtype=torch.complex64, device="cuda")
    op = torch.empty(max(dg.conv_nparts, 1) * 2, dtype=torch.float64, device="cuda")
    nat.check(L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(),
                              nat.stream_handle()), "conv")
    torch.cuda.synchronize()
    pc = u.view(torch.int64).flatten()[: 148 * 12].cpu().numpy().reshape(-1, 12)
    names = ["prod_wait_empty", "1", "2", "mma_wait_full", "mma_wait_tempty", "mma_commit", "epi_wait_tfull",
             "epi_drain", "start", "total", "epi_window", "11"]
    print(json.dumps({n: int(np.median(pc[:, i])) for i, n in enumerate(names) if not n.isdigit() and n != "start"}))
    print("even CTAs", json.dumps({n: int(np.median(pc[0::2, i])) for i, n in enumerate(names) if not n.isdigit() and n != "start"}))
    print("odd CTAs", json.dumps({n: int(np.median(pc[1::2, i])) for i, n in enumerate(names) if not n.isdigit() and n != "start"}))
