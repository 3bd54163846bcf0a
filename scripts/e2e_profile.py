"""cProfile of one end-to-end hicu_reconstruct call (after warm-up): python scripts/e2e_profile.py [C1|C2|C4|C5]."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H
from paper_2004_08962_b200.synthetic import CONFIGS, make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = CONFIGS[name]
ksp, mask, x0 = make_config(name)
cc = spec.coils_out if spec.coils_out != spec.coils_in else None
kern = H.KernelMask.full(spec.kernel)
sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=0)
for _ in range(2):
    H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=cc)
t = time.perf_counter()
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=cc)
print("e2e ms", 1e3 * (time.perf_counter() - t))
pr = cProfile.Profile()
pr.enable()
H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=cc)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
