"""End-to-end golden fixtures produced by running the REFERENCE's own
``hicu.hicu_reconstruct`` (pkg/src/hicu/solver.py:258-398) on the
BASELINE.json synthetic configs.

Run in the build container (where /root/reference exists), one case per
process (they are independent; C2 takes a few CPU minutes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_e2e.py c1
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_e2e.py c2
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_e2e.py c2lock
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_e2e.py c4lock

Inputs are regenerated on the GPU box from the repo's seeded generators
(``paper_2004_08962_b200.synthetic.make_config``) and, for the coil-compressed
configs, the coil basis stored here; norms of the inputs are stored so a test
can detect a drifted generator.  What is stored per case:

* ``c1`` / ``c2``: the reference's free-running reconstruction of the full
  config (C1: 128x128x8, rank 40, 50 iterations; C2: 256x256, 16 coils
  compressed to 8 by the oracle's SVD coil compression, rank 60, 64^2 ->
  128^2 -> full center-out stages, 25/25/50 iterations): per-step SER, eta
  and objective traces, and the final SER.  The device is compared by final
  SER (<= 0.1 dB), because the reference's zgesdd singular-vector phases are
  a LAPACK detail the device cannot reproduce.
* ``c2lock`` / ``c4lock``: short schedules with the reference's V logged at
  every outer iteration (by wrapping ``hicu.solver.rsvd_right_vectors``), the
  eta / objective traces, and the final iterate at a fixed random subset of
  entries: the device, fed the same V, must follow the same trajectory.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("HICU_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import hicu  # noqa: E402  (the reference package)
import hicu.solver as ref_solver  # noqa: E402
from hicu import KernelMask, SolverSchedule, StageSpec, hicu_reconstruct  # noqa: E402

from oracle import hicu_oracle as O  # noqa: E402  (coil compression restatement; the reference has none)
from paper_2004_08962_b200.synthetic import CONFIGS, make_config  # noqa: E402

SUBSET = 65536


def compressed_input(name, scale=1.0):
    """(x0c, maskc, refc, basis) in complex64 after the oracle's SVD coil
    compression of the config's k-space (the input both sides receive)."""
    spec = CONFIGS[name]
    ksp, mask, x0 = make_config(name, scale=scale)
    if spec.coils_out == spec.coils_in:
        return x0, mask, ksp, None
    xc, mc, v = O.coil_compress(x0, mask, spec.coils_out)
    refc = (ksp.astype(np.complex128).reshape(-1, spec.coils_in) @ v).reshape(xc.shape)
    return xc.astype(np.complex64), np.ascontiguousarray(mc), refc.astype(np.complex64), v


def schedule_of(stages, rank, seed=0, circular=()):
    return SolverSchedule(rank=rank, stages=[StageSpec(*s) for s in stages], circular_axes=tuple(circular), seed=seed)


def subset_index(size, seed=1234):
    return np.sort(np.random.default_rng(seed).choice(size, size=min(SUBSET, size), replace=False))


def record(out, x0c, maskc, refc, kernel, sched, report, xhat):
    out["x0_norm"] = np.array(np.linalg.norm(x0c.astype(np.complex128)))
    out["ref_norm"] = np.array(np.linalg.norm(refc.astype(np.complex128)))
    out["mask_sum"] = np.array(int(maskc.sum()))
    out["eta"] = np.array([s.eta for s in report.steps])
    out["obj"] = np.array([s.objective_before for s in report.steps])
    out["obj_after"] = np.array([s.objective_after for s in report.steps])
    out["ser_steps"] = np.array([np.nan if s.ser_db is None else s.ser_db for s in report.steps])
    out["ser_iters"] = np.array([np.nan if i.ser_db is None else i.ser_db for i in report.iterations])
    out["ser_final"] = np.array(O.ser_db(refc, xhat))
    out["ser_zero_filled"] = np.array(O.ser_db(refc, x0c))
    idx = subset_index(xhat.size)
    out["xhat_idx"] = idx.astype(np.int64)
    out["xhat_sub"] = xhat.reshape(-1)[idx]
    out["xhat_norm"] = np.array(np.linalg.norm(xhat))
    out["seconds"] = np.array(report.total_seconds)
    out["meta"] = np.array(json.dumps(dict(
        kernel=list(kernel.extents), rank=sched.rank, seed=sched.seed,
        stages=[[st.region, st.p, st.gradient_steps, st.iterations] for st in sched.stages],
        circular_axes=list(sched.circular_axes), dims=list(x0c.shape), counters=report.counters,
        events=report.events)))


def free_run(name, fname):
    spec = CONFIGS[name]
    x0c, maskc, refc, v = compressed_input(name)
    kernel = KernelMask.full(spec.kernel)
    sched = schedule_of(spec.stages, spec.rank, seed=0, circular=spec.circular_axes)
    t = time.perf_counter()
    xhat, report = hicu_reconstruct(x0c, maskc, kernel, sched, reference=refc, tail_energy_threshold=0)
    out = {}
    record(out, x0c, maskc, refc, kernel, sched, report, xhat)
    if v is not None:
        out["coil_basis"] = v
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(f"{name}: zero-filled {float(out['ser_zero_filled']):.3f} dB -> reference {float(out['ser_final']):.3f} dB "
          f"({time.perf_counter() - t:.0f} s)", flush=True)


def lockstep(name, fname, stages, scale=1.0, v_dtype=np.complex128):
    spec = CONFIGS[name]
    x0c, maskc, refc, v = compressed_input(name, scale=scale)
    kernel = KernelMask.full(spec.kernel)
    sched = schedule_of(stages, spec.rank, seed=0)
    vlog = []
    orig = ref_solver.rsvd_right_vectors

    def logged(*a, **k):
        vv = orig(*a, **k)
        vlog.append(np.array(vv))
        return vv

    ref_solver.rsvd_right_vectors = logged
    try:
        t = time.perf_counter()
        xhat, report = hicu_reconstruct(x0c, maskc, kernel, sched, reference=refc, tail_energy_threshold=0)
    finally:
        ref_solver.rsvd_right_vectors = orig
    out = {}
    record(out, x0c, maskc, refc, kernel, sched, report, xhat)
    out["v_log"] = np.stack(vlog).astype(v_dtype)
    out["scale"] = np.array(scale)
    if v is not None:
        out["coil_basis"] = v
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(f"{name} lockstep ({len(vlog)} iterations, {time.perf_counter() - t:.0f} s)", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c2lock", "c4lock"]
    for w in which:
        if w == "c1":
            free_run("C1", "golden_e2e_c1.npz")
        elif w == "c2":
            free_run("C2", "golden_e2e_c2.npz")
        elif w == "c2lock":
            lockstep("C2", "golden_lock_c2.npz",
                     [([64, 64], 8, 5, 2), ([128, 128], 8, 5, 2), ("full", 8, 5, 2)])
        elif w == "c4lock":
            # C4's 5x5x5x8 kernel (n = 1000) at rank 150 (l = 225) on a 24x18x25
            # series (scale 1/8 in x/y, all 25 frames, 12 -> 8 coils):
            # center-out [16, 12, full] stage then the full grid
            lockstep("C4", "golden_lock_c4.npz", [([16, 12, "full"], 8, 5, 1), ("full", 8, 5, 1)], scale=0.125,
                     v_dtype=np.complex64)
        else:
            raise SystemExit(f"unknown case {w}")
