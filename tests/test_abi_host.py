"""CPU-only checks: the C-ABI library loads and exports every declared
symbol; host-side logic (stage regions, validation, RNG streams) matches the
reference's golden values.  No GPU compute here."""

import json
import os
import re

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import _native as nat
from paper_2004_08962_b200.solver import draw_stage
from oracle import hicu_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hicu_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hicu_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(nat.LIB_PATH):
        from paper_2004_08962_b200 import _build

        _build.build()
    return nat.load()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table binds exactly what the header declares
    assert sorted(nat.EXPORTED) == syms


def test_library_info_without_gpu(lib):
    assert lib.hicu_abi_version() == 2
    assert lib.hicu_status_string(3) == b"DegenerateInputError"
    assert lib.hicu_status_string(6) == b"ConfigError"


def test_struct_layout_matches_header(lib):
    import ctypes

    # hicu_geom: 2*int32 + 3*8*int64 + uint32 (+pad) + 2 pointers
    assert ctypes.sizeof(nat.HicuGeom) == 8 + 3 * 64 + 8 + 16 + 64
    assert nat.HicuStageArgs.rec.offset % 8 == 0


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.NativeError):
        H.hankel_apply(np.ones((4, 4, 2)), np.ones((8, 1)), H.KernelMask.full((2, 2, 2)),
                       H.full_region((4, 4, 2), H.KernelMask.full((2, 2, 2))))


def test_stage_region_matches_reference_table(golden_ops):
    for row in json.loads(str(golden_ops["stage_table"])):
        reg = H.stage_region(tuple(row["dims"]), H.KernelMask.full(row["kext"]), row["frac"], tuple(row["circ"]))
        assert list(reg.offsets) == row["offsets"] and list(reg.extents) == row["extents"], row


def test_stage_region_errors():
    k = H.KernelMask.full((5, 5, 2))
    with pytest.raises(H.ConfigError):
        H.stage_region((16, 16, 2), k, [0.125, 0.5])
    with pytest.raises(H.ConfigError):
        H.stage_region((16, 16, 2), k, [1.5])
    with pytest.raises(H.ConfigError):
        H.stage_region((16, 16, 2), k, [True])
    with pytest.raises(H.ConfigError):
        H.stage_region((16, 16, 2), k, [0.5, 0.5, 0.5, 0.5])


def test_schedule_validation():
    k = H.KernelMask.full((3, 3, 2))
    dims = (10, 10, 2)
    with pytest.raises(H.ConfigError):
        H.SolverSchedule(rank=k.n, stages=[H.StageSpec("full", 1, 1, 1)]).validate(k, dims)
    with pytest.raises(H.ConfigError):
        H.SolverSchedule(rank=3, stages=[]).validate(k, dims)
    with pytest.raises(H.ConfigError):
        H.SolverSchedule(rank=3, stages=[H.StageSpec("full", 0, 1, 1)]).validate(k, dims)
    with pytest.raises(H.ConfigError):
        H.SolverSchedule(rank=3, stages=[H.StageSpec("full", 1, 1, 1)], dc_mode="soft").validate(k, dims)
    with pytest.raises(H.ConfigError):
        H.hicu_reconstruct(np.zeros(dims), np.zeros((10, 9, 2)), k,
                           H.SolverSchedule(rank=3, stages=[H.StageSpec("full", 1, 1, 1)]))


def test_kernel_and_region_errors():
    with pytest.raises(H.ShapeError):
        H.KernelMask((0, 3))
    with pytest.raises(H.ShapeError):
        H.full_region((3,), H.KernelMask.full((5,)))
    with pytest.raises(H.ShapeError):
        H.Region((0,), (0,))
    k = H.KernelMask.ellipsoid((5, 5))
    assert k.n < 25 and k.support[2, 2] == 1 and k.support[0, 0] == 0


def test_rng_streams_match_oracle():
    sched = H.SolverSchedule(rank=6, stages=[H.StageSpec("full", 3, 2, 2)], seed=9)
    omega, pbig = draw_stage(sched, 0, sched.stages[0], 20)
    for it in range(2):
        ref_om = O.complex_normal(O.rng_generator(9, (1, 0, it)), (20, 9))
        assert np.array_equal(omega[it], ref_om)
        for j in range(2):
            P = O.complex_normal(O.rng_generator(9, (2, 0, it, j)), (14, 3), 1.0 / 3)
            assert np.array_equal(pbig[it, 6:, j * 3:(j + 1) * 3], P)
            assert not np.any(pbig[it, :6])


def test_golden_sketch_stream(golden_ops):
    g = golden_ops
    om = H.complex_normal(H.RngStream(int(g["sub_seed"]), tuple(int(i) for i in g["sub_ids"])).generator(),
                          (75, 18))
    assert np.array_equal(om, g["sub_omega"])


def test_mask_apply_bit_exact():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((6, 5)) + 1j * rng.standard_normal((6, 5))
    m = (rng.random((6, 5)) < 0.5).astype(np.uint8)
    y = H.mask_apply(x, m)
    assert np.array_equal(y[m == 1], x[m == 1]) and not np.any(y[m == 0])


def test_report_serializable():
    r = H.ReconReport()
    r.steps.append(H.StepRecord(0, 0, 0, 1.0, 2.0, 1.0, 0.1, float("inf")))
    r.iterations.append(H.IterationRecord(0, 0, 1.0, 0.1))
    json.dumps(r.to_dict())
