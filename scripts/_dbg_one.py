import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry
dims = (70, 300, 8)
kernel = H.KernelMask.full((5, 5, 8)); region = H.full_region(dims, kernel)
dg = device_geometry(kernel, region, dims); L = nat.lib(); st = nat.stream_handle()
y = torch.randn(dims, dtype=torch.complex64, device="cuda"); q = torch.randn((200, 8), dtype=torch.complex64, device="cuda")
u = torch.zeros((dg.s, 8), dtype=torch.complex64, device="cuda"); op = torch.zeros(dg.conv_nparts * 2, dtype=torch.float64, device="cuda")
nat.check(L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(), st))
torch.cuda.synchronize()
print("ok")
import os
if os.environ.get("HICU_CONV_TC_DEBUG") == "32":
    t = u.view(torch.int32).cpu().numpy().reshape(-1)[:200]
    print("ngroups", t[0], t[1:1 + 6 * min(t[0], 30)].reshape(-1, 6).tolist())
