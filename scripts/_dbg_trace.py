import os, sys, json
os.environ["HICU_CONV_TC_DEBUG"] = sys.argv[1] if len(sys.argv) > 1 else "16"
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry
for dims in [(256, 256, 8), (64, 64, 8)]:
    kernel = H.KernelMask.full((5, 5, 8)); region = H.full_region(dims, kernel)
    dg = device_geometry(kernel, region, dims); L = nat.lib(); st = nat.stream_handle()
    y = torch.randn(dims, dtype=torch.complex64, device="cuda"); q = torch.randn((200, 8), dtype=torch.complex64, device="cuda")
    u = torch.zeros((dg.s, 8), dtype=torch.complex64, device="cuda"); op = torch.zeros(dg.conv_nparts * 2, dtype=torch.float64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        nat.check(L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(), st))
        torch.cuda.synchronize()
    t = u.view(torch.int64).cpu().numpy().reshape(-1)[: 148 * 12].reshape(148, 12)[:, :12].astype(np.int64)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t - base) / 1000.0
    print(dims, "ctas", len(t), "us rel to first start: median per milestone", np.round(np.median(rel, axis=0), 2).tolist(),
          "max", np.round(rel.max(axis=0), 2).tolist())
