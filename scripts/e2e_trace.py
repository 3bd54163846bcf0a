"""Host phase marks of one hicu_reconstruct call (HICU_E2E_TRACE=1) at a
config's full size, after a warm-up call."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ["HICU_E2E_TRACE"] = "1"
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
spec = CONFIGS[name]
ksp, mask, x0 = make_config(name)
kern = H.KernelMask.full(spec.kernel)
sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=0)
cc = None if spec.coils_in == spec.coils_out else spec.coils_out
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=cc)
print("---- timed call", file=sys.stderr)
t = time.perf_counter()
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=cc)
print(f"{name} e2e call {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr)
