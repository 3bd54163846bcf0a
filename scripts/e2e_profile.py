"""cProfile of one end-to-end C2 hicu_reconstruct call (after warm-up)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

spec = CONFIGS["C2"]
ksp, mask, x0 = make_config("C2")
kern = H.KernelMask.full(spec.kernel)
sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=0)
for _ in range(2):
    H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=8)
t = time.perf_counter()
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=8)
print("e2e ms", 1e3 * (time.perf_counter() - t))
pr = cProfile.Profile()
pr.enable()
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=8)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
