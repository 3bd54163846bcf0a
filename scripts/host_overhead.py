"""Host-side cost per ABI launch (no synchronisation inside the timed loop)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry

dims = (256, 256, 8)
kernel = H.KernelMask.full((5, 5, 8))
region = H.full_region(dims, kernel)
dg = device_geometry(kernel, region, dims)
L = nat.lib()
st = nat.stream_handle()
y = torch.randn(dims, dtype=torch.complex64, device="cuda")
q = torch.randn((200, 8), dtype=torch.complex64, device="cuda")
u = torch.empty((dg.s, 8), dtype=torch.complex64, device="cuda")
op = torch.empty(dg.conv_nparts * 2, dtype=torch.float64, device="cuda")
rec = torch.zeros(8, dtype=torch.float64, device="cuda")
calls = {
    "conv_fwd": lambda: L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(), st),
    "step_update": lambda: L.hicu_step_update(y.numel(), y.data_ptr(), y.data_ptr(), op.data_ptr(), 1, op.data_ptr(), 1,
                                              op.data_ptr(), 1, 0, 0.0, rec.data_ptr(), st),
    "timestamp": lambda: L.hicu_timestamp(rec.data_ptr(), st),
}
for name, f in calls.items():
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    n = 300
    t = time.perf_counter()
    for _ in range(n):
        f()
    dt = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    print(f"{name}: {dt * 1e6:.1f} us host per call (incl. ctypes)")
