"""Time the Gram paths on one config geometry (default: the full C5 volume):
lag (default) vs dense tcgen05, CUDA events, best of 3 (the workspace
allocation inside gram_matrix is included).  Under ncu it gives the
per-kernel launch list of the lag Gram."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.subspace import gram_matrix
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
paths = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lag", "tcgen05"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec = CONFIGS[name]
ksp, mask, x0 = make_config(name)
x = torch.as_tensor(ksp[..., :spec.coils_out].astype(np.complex64)).cuda()
k = H.KernelMask.full(tuple(spec.kernel[:-1]) + (spec.coils_out,))
reg = H.stage_region(tuple(x.shape), k, spec.stages[-1][0])
for path in paths:
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gram_matrix(x, k, reg, path=None if path == "lag" else path)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name} Gram {path}: {best:.2f} ms (s = {reg.s}, n = {k.n})", flush=True)
