"""Time the tcgen05 conv / scatter at the C5 volume geometry (256x160x160x8,
5x5x5x8 kernel, p = 8) with CUDA events; HICU_CONV_TC_DEBUG (read once per
process) switches parts off for a bound split: 1 no MMA, 2 no TMA, 4 no
hi/lo conversion, 8 no TMEM drain.  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256,160,160,8").split(","))
kext = (5, 5, 5, 8) if len(dims) == 4 else (5, 5, 8)
kernel = H.KernelMask.full(kext)
region = H.full_region(dims, kernel)
dg = device_geometry(kernel, region, dims)
L = nat.lib()
g = torch.Generator(device="cuda").manual_seed(0)
y = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
mask = (torch.rand(dims, device="cuda", generator=g) < 0.25).to(torch.uint8)
q = torch.randn((kernel.n, 8), dtype=torch.complex64, device="cuda", generator=g) / kernel.n ** 0.5
u = torch.randn((dg.s, 8), dtype=torch.complex64, device="cuda", generator=g)
gout = torch.empty(dims, dtype=torch.complex64, device="cuda")
op = torch.empty(max(dg.conv_nparts, 1) * 2, dtype=torch.float64, device="cuda")
sp = torch.empty(max(dg.scatter_nparts, 1) * 4, dtype=torch.float64, device="cuda")
calls = {
    "conv_fwd": lambda: L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(),
                                        nat.stream_handle()),
    "scatter_hard": lambda: L.hicu_scatter_dc(dg.ref(), q.data_ptr(), 8, u.data_ptr(), mask.data_ptr(), None, None,
                                              0, 0.0, gout.data_ptr(), sp.data_ptr(), nat.stream_handle()),
}
out = {"debug": int(os.environ.get("HICU_CONV_TC_DEBUG", "0")), "dims": list(dims)}
for name, f in calls.items():
    for _ in range(3):
        nat.check(f(), name)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        nat.check(f(), name)
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = round(e0.elapsed_time(e1) / 5, 3)
print(json.dumps(out), flush=True)
