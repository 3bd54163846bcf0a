"""Throughput of independent C2 reconstructions run concurrently on CUDA
streams (hicu_reconstruct_batch), end to end from host arrays."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2004_08962_b200 as H
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

spec = CONFIGS["C2"]
kern = H.KernelMask.full(spec.kernel)
sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=0)
data = [make_config("C2", slice_index=i) for i in range(8)]
x0s, masks = [d[2] for d in data], [d[1] for d in data]
out = {}
for conc in (1, 2, 4, 8):
    n = 8
    H.hicu_reconstruct_batch(x0s[:conc], masks[:conc], kern, sched, concurrency=conc, tail_energy_threshold=0,
                             coil_compress=8)
    torch.cuda.synchronize()
    t = time.perf_counter()
    H.hicu_reconstruct_batch(x0s[:n], masks[:n], kern, sched, concurrency=conc, tail_energy_threshold=0,
                             coil_compress=8)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out[conc] = {"slices": n, "s": round(dt, 3), "iters_per_s": round(n * spec.iterations / dt, 1)}
print(json.dumps(out))
