"""Does capturing a whole reconstruction in a CUDA graph help the launch-heavy
small configs?  Eager (PDL launches from the native stage driver) against a
replayed graph of the same run_all(), C1 or C2, device-resident, CUDA events.
usage: python scripts/graph_probe.py [C1|C2]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.coil import coil_compress_device
from paper_2004_08962_b200.hankel import to_dev
from paper_2004_08962_b200.solver import ReconEngine, draw_stage
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
spec = CONFIGS[name]
ksp, mask, x0 = make_config(name)
kern = H.KernelMask.full(spec.kernel)
sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=0)
xd = to_dev(x0).reshape(-1)
md = to_dev(mask, np.uint8).reshape(-1)
nc, nv = spec.coils_in, spec.coils_out
if nv != nc:
    y, m, _, _ = coil_compress_device(xd, md, nc, nv)
else:
    y, m = xd, md
dims = x0.shape[:-1] + (nv,)
regions = sched.validate(kern, dims)
eng = ReconEngine(y, m, dims, kern, sched, regions)
for si, st in enumerate(sched.stages):
    om, pb = draw_stage(sched, si, st, kern.n)
    eng.set_host_draws(si, om, pb)
x_init = eng.x_init.clone()


def once():
    eng.y.copy_(x_init)
    eng.status.zero_()
    eng.run_all()


def timed(f, reps=5):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0.record()
        f()
        host = time.perf_counter() - t
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, host * 1e3


for _ in range(3):
    once()
torch.cuda.synchronize()
ref = eng.y.clone()
ms, host = timed(once)
print(f"{name} eager: {ms:.2f} ms device, {host:.2f} ms host issue")
try:
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        once()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            once()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(eng.y, ref))
    ms2, host2 = timed(g.replay)
    print(f"{name} graph replay: {ms2:.2f} ms device, {host2:.2f} ms host issue, bit-identical result: {same}")
except Exception as e:  # noqa: BLE001
    print(f"{name} graph capture failed: {type(e).__name__}: {str(e)[:300]}")
