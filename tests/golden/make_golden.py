"""Generate the golden fixtures in this directory by running the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``hicu`` (read-only) and records inputs and
outputs of the hot-path functions on small seeded instances into
``golden_ops.npz`` and ``golden_recon.npz``.  The GPU box never reads
/root/reference; tests only read these committed .npz files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("HICU_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import hicu  # noqa: E402  (the reference package)
from hicu import (  # noqa: E402
    DataConsistency,
    KernelMask,
    MaskSpec,
    PhantomSpec,
    Region,
    SolverSchedule,
    StageSpec,
    exact_line_search,
    full_region,
    gen_mask,
    gen_phantom,
    hankel_adjoint_apply,
    hankel_apply,
    hicu_reconstruct,
    kspace_adjoint_scatter,
    mask_apply,
    numerical_rank,
    objective_and_gradient,
    stage_region,
)
from hicu.subspace import RngStream, householder_nullspace, jl_compress, rsvd_right_vectors  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _rand(g, shape):
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


def _geom_record(prefix, out, dims, kernel, region):
    out[prefix + "dims"] = np.array(dims, np.int64)
    out[prefix + "kext"] = np.array(kernel.extents, np.int64)
    out[prefix + "support"] = kernel.support.astype(np.uint8)
    out[prefix + "roff"] = np.array(region.offsets, np.int64)
    out[prefix + "rext"] = np.array(region.extents, np.int64)
    circ = np.zeros(len(dims), np.uint8)
    for a in region.circular_axes:
        circ[a] = 1
    out[prefix + "circ"] = circ


def ops_cases():
    out = {}
    cases = [
        # name, dims, kernel extents, circular axes, support kind, region override
        ("c2d", (9, 8, 3), (3, 3, 3), (), "full", None),
        ("c2dcirc", (8, 7, 2), (3, 2, 2), (0, 1), "full", None),
        ("csub", (10, 9, 3), (3, 3, 3), (), "full", ((2, 1, 0), (4, 5, 1))),
        ("c3d", (6, 5, 4, 2), (3, 2, 2, 2), (2,), "full", None),
        ("cell", (9, 9, 2), (5, 5, 2), (), "ellipsoid", None),
        ("c1d", (12,), (4,), (), "full", None),
        ("cnc", (8, 8, 4), (3, 3, 1), (), "full", None),   # kernel narrower than coil axis
    ]
    names = []
    for ci, (name, dims, kext, circ, kind, reg_override) in enumerate(cases):
        g = np.random.default_rng(100 + ci)
        kernel = KernelMask.ellipsoid(kext) if kind == "ellipsoid" else KernelMask.full(kext)
        if reg_override is None:
            region = full_region(dims, kernel, circ)
        else:
            region = Region(reg_override[0], reg_override[1], frozenset(circ))
            region.validate(kernel, dims)
        p = f"{name}_"
        _geom_record(p, out, dims, kernel, region)
        x = _rand(g, dims)
        v = _rand(g, (kernel.n, 3))
        u = _rand(g, (region.s, 3))
        out[p + "x"] = x
        out[p + "v"] = v
        out[p + "u"] = u
        out[p + "fwd"] = hankel_apply(x, v, kernel, region)
        out[p + "adj"] = hankel_adjoint_apply(x, u, kernel, region)
        out[p + "scatter"] = kspace_adjoint_scatter(v, u, kernel, region, dims)
        out[p + "gram"] = hankel_adjoint_apply(x, hankel_apply(x, np.eye(kernel.n), kernel, region),
                                               kernel, region)
        mask = (g.random(dims) < 0.4).astype(np.uint8)
        x0 = mask_apply(_rand(g, dims), mask)
        out[p + "mask"] = mask
        out[p + "x0"] = x0
        for mode in ("hard", "soft"):
            dc = DataConsistency(mode, mask, x0=x0 if mode == "soft" else None,
                                 lam=0.7 if mode == "soft" else 0.0)
            grad, obj, uu = objective_and_gradient(x, v, kernel, region, dc, return_products=True)
            eta, dec = exact_line_search(x, grad, v, kernel, region, dc, u=uu, return_decrease=True)
            out[p + mode + "_grad"] = grad
            out[p + mode + "_obj"] = np.array(obj)
            out[p + mode + "_eta"] = np.array(eta)
            out[p + mode + "_dec"] = np.array(dec)
        names.append(name)
    out["op_cases"] = np.array(names)

    # subspace: rSVD, Householder, JL on a phantom-like instance
    spec = PhantomSpec(nx=16, ny=16, ncoils=3, sens_kspace_order=1, seed=5)
    ksp, _ = gen_phantom(spec)
    g = np.random.default_rng(7)
    ksp = ksp + 1e-3 * np.abs(ksp).max() * _rand(g, ksp.shape)
    kernel = KernelMask.full((5, 5, 3))
    region = full_region(ksp.shape, kernel)
    out["sub_x"] = ksp
    out["sub_kext"] = np.array(kernel.extents)
    out["sub_rank"] = np.array(12)
    out["sub_seed"] = np.array(3)
    out["sub_ids"] = np.array([1, 0, 2])
    v = rsvd_right_vectors(ksp, kernel, region, 12, RngStream(3, (1, 0, 2)))
    out["sub_v"] = v
    q = householder_nullspace(v).q
    out["sub_q"] = q
    out["sub_qt"] = jl_compress(q, 4, RngStream(3, (2, 0, 2, 1)))
    out["sub_omega"] = hicu.subspace.complex_normal(RngStream(3, (1, 0, 2)).generator(), (kernel.n, 18), 1.0)

    # stage_region table (solver.py:127-158), incl. banker's rounding
    table = []
    for dims, kext, frac, circ in [
        ((384, 384, 8), (5, 5, 8), "full", ()),
        ((384, 384, 8), (5, 5, 8), [0.25, 0.25], ()),
        ((64, 64, 16, 8), (5, 5, 3, 8), [0.25, 0.25, 0.25], (2,)),
        ((32, 32, 4), (5, 5, 4), [0.5, 0.5, 0.5], ()),
        ((20, 20, 2), (3, 3, 2), [8, "full"], ()),
        ((256, 256, 8), (5, 5, 8), [64, 64], ()),
        ((256, 256, 8), (5, 5, 8), [128, 128], ()),
        ((192, 144, 25, 8), (5, 5, 5, 8), [48, 36, "full"], ()),
        ((20, 20, 2), (3, 3, 2), [0.225, 0.175], ()),  # round(4.5)=4, round(3.5)=4
        ((30, 30, 2), (3, 3, 2), [0.5, 0.15], ()),    # round(15.0), round(4.5)=4
    ]:
        reg = stage_region(dims, KernelMask.full(kext), frac, circ)
        table.append(dict(dims=list(dims), kext=list(kext), frac=frac, circ=list(circ),
                          offsets=list(reg.offsets), extents=list(reg.extents)))
    out["stage_table"] = np.array(json.dumps(table))
    np.savez_compressed(os.path.join(HERE, "golden_ops.npz"), **out)


def _run(out, meta, name, sched, x0, mask, ksp, kernel, data):
    xhat, report = hicu_reconstruct(x0, mask, kernel, sched, reference=ksp, tail_energy_threshold=0)
    out[name + "_xhat"] = xhat
    out[name + "_eta"] = np.array([s.eta for s in report.steps])
    out[name + "_obj"] = np.array([s.objective_before for s in report.steps])
    out[name + "_obj_after"] = np.array([s.objective_after for s in report.steps])
    out[name + "_ser"] = np.array([s.ser_db for s in report.steps])
    meta[name] = dict(rank=sched.rank, seed=sched.seed, dc_mode=sched.dc_mode,
                      dc_lambda=sched.dc_lambda, circular_axes=list(sched.circular_axes),
                      stages=[[st.region, st.p, st.gradient_steps, st.iterations]
                              for st in sched.stages],
                      counters=report.counters, events=report.events, data=data)


def recon_case():
    spec = PhantomSpec(nx=20, ny=20, ncoils=3, sens_kspace_order=1, seed=21)
    ksp, _ = gen_phantom(spec)
    g = np.random.default_rng(22)
    ksp = ksp + 3e-3 * np.linalg.norm(ksp) / np.sqrt(ksp.size) * _rand(g, ksp.shape)
    mask = gen_mask(ksp.shape, MaskSpec("vd_1d", 2.0, acs=(4,), seed=15, vd_decay=1.0, vd_sigma_frac=0.5))
    x0 = mask_apply(ksp, mask)
    kernel = KernelMask.full((5, 5, 3))
    out = {"x0": x0, "mask": mask, "ref": ksp, "kext": np.array(kernel.extents)}
    # short runs pin trajectories (lockstep parity) on the problem above
    runs = {
        "hard": SolverSchedule(rank=20, stages=[StageSpec([12, 12], 3, 3, 2), StageSpec("full", 4, 3, 3)],
                               seed=5),
        "soft": SolverSchedule(rank=20, stages=[StageSpec("full", 3, 2, 3)], dc_mode="soft",
                               dc_lambda=5.0, seed=6),
        "circ": SolverSchedule(rank=20, stages=[StageSpec("full", 3, 3, 3)], circular_axes=(0, 1), seed=7),
    }
    meta = {}
    for name, sched in runs.items():
        _run(out, meta, name, sched, x0, mask, ksp, kernel, "base")

    # long runs: a problem HICU actually solves (the reference's own recovery
    # test problem, pkg/tests/test_solver.py:24-35 + 128-141, with 1 % noise so
    # the fp32 device and the fp64 reference converge to the same noise
    # floor): 24x24x3, numerical rank 49, vd_1d R=1.6.  Zero-filled SER
    # 15.7 dB; the reference reaches 23.6 / 29.1 / 20.4 dB (hard / circular /
    # soft), so the final SER does not depend on the singular-vector phase
    # convention to within ~0.06 dB and can be compared with the device's.
    spec = PhantomSpec(nx=24, ny=24, ncoils=3, sens_kspace_order=1, seed=7)
    ksp2, _ = gen_phantom(spec)
    kern2 = KernelMask.full((5, 5, 3))
    rank2 = int(numerical_rank(ksp2, kern2, full_region(ksp2.shape, kern2, (0, 1))))
    g = np.random.default_rng(22)
    ksp2 = ksp2 + 1e-2 * np.linalg.norm(ksp2) / np.sqrt(ksp2.size) * _rand(g, ksp2.shape)
    mask2 = gen_mask(ksp2.shape, MaskSpec("vd_1d", 1.6, acs=(4,), seed=15, vd_decay=1.0, vd_sigma_frac=0.5))
    lx0 = mask_apply(ksp2, mask2)
    out["lp_x0"], out["lp_mask"], out["lp_ref"], out["lp_kext"] = lx0, mask2, ksp2, np.array(kern2.extents)
    long_runs = {
        "hardlong": SolverSchedule(rank=rank2, stages=[StageSpec([18, 18], 3, 5, 10), StageSpec("full", 12, 10, 30)],
                                   seed=4),
        "circlong": SolverSchedule(rank=rank2, stages=[StageSpec("full", 3, 5, 10), StageSpec("full", 12, 10, 30)],
                                   circular_axes=(0, 1), seed=4),
        "softlong": SolverSchedule(rank=rank2, stages=[StageSpec("full", 6, 5, 20)], dc_mode="soft",
                                   dc_lambda=5.0, seed=4),
    }
    for name, sched in long_runs.items():
        _run(out, meta, name, sched, lx0, mask2, ksp2, kern2, "lp")
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "golden_recon.npz"), **out)


if __name__ == "__main__":
    ops_cases()
    recon_case()
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))
