"""Time hicu_gram (C2 stage geometries) with CUDA-graph replays and check it
against the SIMT Gram; prints one JSON line.  HICU_GRAM_GATHER=1 selects the
gather-producer tcgen05 kernel instead of the TMA-fed one."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry


def run(dims, window, reps=50, kext=(5, 5, 8)):
    kernel = H.KernelMask.full(kext)
    if window is None:
        region = H.full_region(dims, kernel)
    else:
        off = tuple((d - window) // 2 for d in dims[:2]) + (0,)
        region = H.Region(off, (window - 4, window - 4, 1), frozenset())
    uses_tc = bool(nat.lib().hicu_gram_uses_tensor_cores(device_geometry(kernel, region, dims).ref()))
    dg = device_geometry(kernel, region, dims)
    L = nat.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    ws_bytes = L.hicu_gram_workspace(dg.ref())
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    G = torch.empty((kernel.n, kernel.n), dtype=torch.complex128, device="cuda")
    f = lambda st: L.hicu_gram(dg.ref(), x.data_ptr(), G.data_ptr(), ws.data_ptr(), ws_bytes, st)
    nat.check(f(nat.stream_handle()), "gram")
    torch.cuda.synchronize()
    Gs = H.gram_matrix(x, kernel, region, force_simt=True)
    err = float((G - Gs).abs().max() / Gs.abs().max())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st = nat.stream_handle()
        for _ in range(reps):
            nat.check(f(st), "gram")
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    s = region.s
    flops = 4 * s * kernel.n * (kernel.n + 1)
    return {"rows": s, "n": kernel.n, "tcgen05": uses_tc, "us": round(us, 2), "tflops": round(flops / us / 1e6, 2),
            "rel_err_vs_simt": err}


if __name__ == "__main__":
    out = {}
    for tag, dims, win in [("C2_full", (256, 256, 8), None), ("C2_stage2", (256, 256, 8), 128),
                           ("C2_stage1", (256, 256, 8), 64)]:
        out[tag] = run(dims, win)
    if "--big" in sys.argv:
        # C3 slice (7x7x10 kernel) and the per-GPU shard of C5 (5x5x5x8 kernel, 32 output planes + 4 halo)
        out["C3_slice"] = run((320, 320, 10), None, reps=5, kext=(7, 7, 10))
        out["C5_shard"] = run((36, 160, 160, 8), None, reps=3, kext=(5, 5, 5, 8))
    print(json.dumps(out))
