"""Time conv_fwd / conv_els / scatter_dc (C2 stage geometries, p = 8) on the
tcgen05 path vs the SIMT path with CUDA events, and report each path's error
against the oracle at C2 full size; prints one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from oracle import hicu_oracle as O
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.hankel import device_geometry


def run(dims, kext, reps=200, simt=False, graph_capture=True):
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    with H.kernel_paths(simt_conv=simt):
        dg = device_geometry(kernel, region, dims)
    L = nat.lib()
    st = nat.stream_handle()
    g = torch.Generator(device="cuda").manual_seed(0)
    y = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    gd = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    x0 = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    mask = (torch.rand(dims, device="cuda", generator=g) < 0.25).to(torch.uint8)
    q = torch.randn((kernel.n, 8), dtype=torch.complex64, device="cuda", generator=g) / kernel.n ** 0.5
    u = torch.empty((dg.s, 8), dtype=torch.complex64, device="cuda")
    gout = torch.empty(dims, dtype=torch.complex64, device="cuda")
    op = torch.empty(max(dg.conv_nparts, 1) * 2, dtype=torch.float64, device="cuda")
    sp = torch.empty(max(dg.scatter_nparts, 1) * 4, dtype=torch.float64, device="cuda")
    calls = {
        "conv_fwd": lambda st: L.hicu_conv_fwd(dg.ref(), y.data_ptr(), q.data_ptr(), 8, u.data_ptr(),
                                               op.data_ptr(), st),
        "conv_els": lambda st: L.hicu_conv_els(dg.ref(), gd.data_ptr(), q.data_ptr(), 8, u.data_ptr(),
                                               op.data_ptr(), st),
        "scatter_soft": lambda st: L.hicu_scatter_dc(dg.ref(), q.data_ptr(), 8, u.data_ptr(), mask.data_ptr(),
                                                     y.data_ptr(), x0.data_ptr(), 1, 0.5, gout.data_ptr(),
                                                     sp.data_ptr(), st),
    }
    out = {}
    for name, f in calls.items():
        for _ in range(5):
            nat.check(f(nat.stream_handle()), name)
        torch.cuda.synchronize()
        if not graph_capture:  # long launches: plain event timing on the stream
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                nat.check(f(nat.stream_handle()), name)
            e1.record()
            torch.cuda.synchronize()
            out[name] = round(e0.elapsed_time(e1) * 1000 / reps, 2)
            continue
        # CUDA-graph replay: GPU time only (no ctypes / host launch overhead)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gst = nat.stream_handle()
            for _ in range(reps):
                nat.check(f(gst), name)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) * 1000 / reps, 2)
    return out, dg.s, kernel.n


def accuracy():
    dims, kext = (256, 256, 8), (5, 5, 8)
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    og = O.Geom(dims, kernel.positions, region.offsets, region.extents, frozenset())
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64).astype(np.complex128)
    q = ((rng.standard_normal((kernel.n, 8)) + 1j * rng.standard_normal((kernel.n, 8))) / 14).astype(
        np.complex64).astype(np.complex128)
    ref = O.hankel_apply(x, q, og)
    gref = O.kspace_adjoint_scatter(q, ref, og)
    rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
    res = {}
    for simt in (False, True):
        with H.kernel_paths(simt_conv=simt):
            res["simt" if simt else "tc"] = {
                "conv_rel_err": rel(H.hankel_apply(x, q, kernel, region), ref),
                "scatter_rel_err": rel(H.kspace_adjoint_scatter(q, ref, kernel, region, dims), gref)}
    return res


if __name__ == "__main__":
    res = {}
    for dims, kext, tag in [((256, 256, 8), (5, 5, 8), "C2_full"), ((128, 128, 8), (5, 5, 8), "C2_stage2"),
                            ((64, 64, 8), (5, 5, 8), "C2_stage1_window")]:
        tc, s, n = run(dims, kext)
        simt, _, _ = run(dims, kext, simt=True)
        flops = 8 * s * n * 8
        res[tag] = {"rows": s, "n": n, "tc_us": tc, "simt_us": simt,
                    "tc_conv_tflops": round(flops / tc["conv_fwd"] / 1e6, 2)}
    res["accuracy_vs_oracle_C2"] = accuracy()
    print(json.dumps(res))
