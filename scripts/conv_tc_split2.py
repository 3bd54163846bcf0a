"""C5 tcgen05 conv / scatter / ELS timing with the engine's prebuilt B images
(the streamed-B production path).  HICU_CONV_TC_DEBUG switches parts off for
a bound split: 1 no MMA, 2 no TMA, 4 no hi/lo conversion, 8 no TMEM drain.
One JSON line."""
import ctypes
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
prep = L._Z24hicu_conv_images_preparePK9hicu_geomPKviiPvmS4_
prep.restype = ctypes.c_size_t
prep.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                 ctypes.c_void_p]
hint = L._Z20hicu_conv_image_hintPKvi
hint.restype = None
hint.argtypes = [ctypes.c_void_p, ctypes.c_int]
g = torch.Generator(device="cuda").manual_seed(0)
y = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
x0 = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
mask = (torch.rand(dims, device="cuda", generator=g) < 0.25).to(torch.uint8)
q = torch.randn((kernel.n, 8), dtype=torch.complex64, device="cuda", generator=g) / kernel.n ** 0.5
u = torch.randn((dg.s, 8), dtype=torch.complex64, device="cuda", generator=g)
gout = torch.empty(dims, dtype=torch.complex64, device="cuda")
op = torch.empty(max(dg.conv_nparts, 1) * 2, dtype=torch.float64, device="cuda")
sp = torch.empty(max(dg.scatter_nparts, 1) * 4, dtype=torch.float64, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
geo = dg.ref()
ib = prep(ctypes.addressof(dg.struct), q.data_ptr(), 8, 1, ws.data_ptr(),
          ws.numel(), nat.stream_handle())
torch.cuda.synchronize()
img = ws.data_ptr()


def with_hint(i, f):
    def run():
        hint(img + i * ib if ib else None, 1)
        r = f()
        hint(None, 0)
        return r
    return run


calls = {
    "conv_fwd": with_hint(0, lambda: L.hicu_conv_fwd(geo, y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(),
                                                     nat.stream_handle())),
    "scatter_soft": with_hint(1, lambda: L.hicu_scatter_dc(geo, q.data_ptr(), 8, u.data_ptr(), mask.data_ptr(),
                                                           y.data_ptr(), x0.data_ptr(), 1, 0.5, gout.data_ptr(),
                                                           sp.data_ptr(), nat.stream_handle())),
    "scatter_hard": with_hint(1, lambda: L.hicu_scatter_dc(geo, q.data_ptr(), 8, u.data_ptr(), mask.data_ptr(), None,
                                                           None, 0, 0.0, gout.data_ptr(), sp.data_ptr(),
                                                           nat.stream_handle())),
    "conv_els": with_hint(0, lambda: L.hicu_conv_els(geo, y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(),
                                                     nat.stream_handle())),
}
out = {"debug": int(os.environ.get("HICU_CONV_TC_DEBUG", "0")), "dims": list(dims), "image_bytes": ib}
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
if out["debug"] & 32:
    # per-role cycle counters of one conv_fwd launch (first 148 x 12 int64 of u)
    hint(img, 1)
    nat.check(L.hicu_conv_fwd(geo, y.data_ptr(), q.data_ptr(), 8, u.data_ptr(), op.data_ptr(), nat.stream_handle()), "c")
    hint(None, 0)
    torch.cuda.synchronize()
    pcs = u.view(torch.int64).flatten()[: 148 * 12].view(148, 12).double().mean(0).tolist()
    names = ["prod_wait_empty", "conv_wait_full", "conv_work", "mma_wait_full", "mma_wait_tempty", "mma_issue",
             "epi_wait_tfull", "epi_drain", "start", "total", "epi_window", "y"]
    out["conv_fwd_cycles"] = {n: round(v) for n, v in zip(names, pcs) if n not in ("start", "y", "conv_wait_full", "conv_work")}
    calls["scatter_hard"]()
    torch.cuda.synchronize()
    pcs = gout.view(torch.int64).flatten()[: 148 * 12].view(148, 12).double().mean(0).tolist()
    out["scatter_cycles"] = {n: round(v) for n, v in zip(names, pcs) if n not in ("start", "y", "conv_wait_full", "conv_work")}
print(json.dumps(out), flush=True)
