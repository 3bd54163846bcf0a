"""Per-GPU workloads of the larger BASELINE configs on one B200, through the
native stage driver (ReconEngine): one C3 slice (320x320, 16->10 coils,
7x7x10 kernel, r=100) and one C5 shard (the 32 readout output planes plus the
4-plane halo that one of 8 GPUs holds: 36x160x160x8, 5x5x5x8 kernel, r=120).
Times `iters` outer iterations (G=5, p=8/10) after one warm-up iteration and
reports ms per iteration, per-kernel-class ms (CUDA-event profiler, one extra
iteration) and the Gram / convolution TFLOP/s.  One JSON line per workload.

Usage: python scripts/shard_bench.py [C3] [C5] [--iters K]"""
import json
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.coil import coil_compress_device
from paper_2004_08962_b200.hankel import to_dev
from paper_2004_08962_b200.solver import ReconEngine, draw_stage
from paper_2004_08962_b200.synthetic import CONFIGS, make_config


def workload(name):
    full = name.endswith("full")
    name = name.replace("full", "")
    spec = CONFIGS[name]
    ksp, mask, x0 = make_config(name)
    if name == "C5" and not full:  # one of 8 shards along readout: 32 output planes + 4 halo planes
        x0, mask = np.ascontiguousarray(x0[:36]), np.ascontiguousarray(mask[:36])
    return spec, x0, mask


def run(name, iters):
    spec, x0, mask = workload(name)
    p = spec.stages[-1][1]
    kernel = H.KernelMask.full(spec.kernel)
    nc, nv = spec.coils_in, spec.coils_out
    xd = to_dev(x0).reshape(-1)
    md = to_dev(mask, np.uint8).reshape(-1)
    y, m, _, _ = coil_compress_device(xd, md, nc, nv)
    dims_c = x0.shape[:-1] + (nv,)
    sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec("full", p, 5, iters + 1)], seed=0)
    regions = sched.validate(kernel, dims_c)
    eng = ReconEngine(y, m, dims_c, kernel, sched, regions)
    om, pb = draw_stage(sched, 0, sched.stages[0], kernel.n)
    eng.set_host_draws(0, om, pb)
    y0 = eng.y.clone()
    # warm-up: all iterations once (loads kernels, sizes workspaces)
    eng.run_all()
    torch.cuda.synchronize()
    eng.check_status()
    eng.y.copy_(y0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run_all()
    e1.record()
    torch.cuda.synchronize()
    eng.check_status()
    ms_it = e0.elapsed_time(e1) / (iters + 1)
    prof = nat.Profiler()
    eng.y.copy_(y0)
    eng.prof = prof
    prof.reset()
    eng.run_all()
    torch.cuda.synchronize()
    eng.prof = None
    kinds = prof.summary()
    s, n = regions[0].s, kernel.n
    it = iters + 1
    gram_f = 4.0 * s * n * (n + 1)
    conv_f = 8.0 * s * n * p  # per conv launch
    k = {kk: v["ms"] / it for kk, v in kinds.items()}
    out = {"workload": name + (" full volume" if len(x0) == 256 else ""), "dims": list(dims_c), "kernel": list(spec.kernel), "n": n, "rank": spec.rank,
           "ell": math.ceil(1.5 * spec.rank), "p": p, "G": 5, "rows": s, "ms_per_iteration": round(ms_it, 3),
           "kernel_ms_per_iteration": {kk: round(v, 3) for kk, v in k.items()},
           "gram_tflops": round(gram_f / (k["gram"] * 1e-3) / 1e12, 2) if k["gram"] else None,
           "conv_fwd_tflops": round(5 * conv_f / (k["conv_fwd"] * 1e-3) / 1e12, 2) if k["conv_fwd"] else None,
           "scatter_tflops": round(5 * conv_f / (k["scatter"] * 1e-3) / 1e12, 2) if k["scatter"] else None,
           "conv_els_tflops": round(5 * conv_f / (k["conv_els"] * 1e-3) / 1e12, 2) if k["conv_els"] else None,
           "gram_tcgen05": bool(nat.lib().hicu_gram_uses_tensor_cores(eng.geoms[0].ref()))
           if hasattr(eng, "geoms") else None}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 2
    if "--iters" in sys.argv:
        args = [a for a in args if a != str(iters)]
    for name in args or ["C3", "C5"]:
        run(name, iters)
