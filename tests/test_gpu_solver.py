"""End-to-end GPU reconstruction behaviour: lockstep trajectory parity with the
oracle's V injected (free-running SER against the reference's own runs lives
in test_gpu_reference_e2e.py), bit-exact hard data consistency, determinism and the
reference solver's behavioural tests (tests/test_solver.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from oracle import hicu_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def sched_from(meta):
    return H.SolverSchedule(rank=meta["rank"], stages=[H.StageSpec(s[0], s[1], s[2], s[3]) for s in meta["stages"]],
                            circular_axes=tuple(meta["circular_axes"]), dc_mode=meta["dc_mode"],
                            dc_lambda=meta["dc_lambda"], seed=meta["seed"])


@pytest.mark.parametrize("name", ["hard", "soft", "circ"])
def test_lockstep_trajectory(golden_recon, name):
    g = golden_recon
    meta = json.loads(str(g["meta"]))[name]
    stages = [tuple(s) for s in meta["stages"]]
    vlog, trace = {}, []
    xo, _ = O.hicu_reconstruct(g["x0"], g["mask"], tuple(g["kext"]), stages, meta["rank"],
                               circular=tuple(meta["circular_axes"]), dc_mode=meta["dc_mode"],
                               dc_lambda=meta["dc_lambda"], seed=meta["seed"], trace=trace, v_log=vlog)
    kern = H.KernelMask.full(tuple(g["kext"]))
    xg, rep = H.hicu_reconstruct(g["x0"], g["mask"], kern, sched_from(meta), tail_energy_threshold=0,
                                 lockstep_v=lambda si, it: vlog[(si, it)])
    eo = np.array([t["eta"] for t in trace])
    eg = np.array([s.eta for s in rep.steps])
    assert np.abs(eg - eo).max() <= 1e-4 * np.abs(eo).max()
    oo = np.array([t["obj"] for t in trace])
    og = np.array([s.objective_before for s in rep.steps])
    assert np.all(np.abs(og - oo) <= 1e-4 * np.abs(oo) + 1e-6 * np.abs(oo).max())
    assert np.linalg.norm(xg - xo) <= 1e-5 * np.linalg.norm(xo)


def _small_problem(seed=7, nx=24, nc=3):
    rng = np.random.default_rng(seed)
    # smooth multi-coil phantom: low-order k-space support -> low-rank lifted matrix
    img = np.zeros((nx, nx), complex)
    yy, xx = np.mgrid[:nx, :nx] / nx - 0.5
    img[(xx / 0.35) ** 2 + (yy / 0.3) ** 2 <= 1] = 1.0
    img[((xx - 0.1) / 0.1) ** 2 + (yy / 0.15) ** 2 <= 1] += 0.5
    sens = np.stack([np.exp(2j * np.pi * (k * xx + (k - 1) * yy) * 0.5) for k in range(nc)], -1)
    ksp = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(img[..., None] * sens, axes=(0, 1)), axes=(0, 1),
                                      norm="ortho"), axes=(0, 1))
    ksp = ksp + 1e-3 * np.abs(ksp).max() * (rng.standard_normal(ksp.shape) + 1j * rng.standard_normal(ksp.shape))
    mask = np.zeros(ksp.shape, np.uint8)
    lines = rng.random(nx) < 0.55
    lines[nx // 2 - 3:nx // 2 + 3] = True
    mask[:, lines, :] = 1
    x0 = np.where(mask == 1, ksp, 0)
    kern = H.KernelMask.full((5, 5, nc))
    return ksp, kern, mask, x0, 20


def test_fully_sampled_identity():
    ksp, kern, _, _, rank = _small_problem()
    ones = np.ones(ksp.shape, np.uint8)
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=2, gradient_steps=2, iterations=2)], seed=1)
    xhat, report = H.hicu_reconstruct(ksp, ones, kern, sched, tail_energy_threshold=0)
    assert np.array_equal(xhat, ksp)
    assert len(report.events) == 4


def test_hard_dc_every_iterate_and_determinism():
    ksp, kern, mask, x0, rank = _small_problem()
    obs = mask == 1
    flags = []
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=3, gradient_steps=3, iterations=4)],
                             circular_axes=(0, 1), seed=2)
    a, _ = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0,
                              iterate_callback=lambda s, i, x: flags.append(np.array_equal(x[obs], x0[obs])))
    assert len(flags) == 4 and all(flags)
    b, _ = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    assert np.array_equal(a, b)
    c, _ = H.hicu_reconstruct(x0, mask, kern, H.SolverSchedule(rank=rank, stages=sched.stages,
                                                               circular_axes=(0, 1), seed=3),
                              tail_energy_threshold=0)
    assert not np.array_equal(a, c)


def test_recovery_improves_ser_and_monotone_objective():
    ksp, kern, mask, x0, rank = _small_problem()
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=3, gradient_steps=5, iterations=10),
                                                H.StageSpec("full", p=12, gradient_steps=10, iterations=10)],
                             circular_axes=(0, 1), seed=4)
    xhat, rep = H.hicu_reconstruct(x0, mask, kern, sched, reference=ksp, tail_energy_threshold=0)
    assert O.ser_db(ksp, xhat) >= O.ser_db(ksp, x0) + 10.0
    assert len(rep.iterations) == 20
    for rec in rep.steps:
        assert rec.objective_after <= rec.objective_before * (1 + 1e-6) + 1e-12
    c = rep.counters
    assert c["gram"] == 20 and c["kspace_scatter"] == 3 * 5 * 10 + 12 * 10 * 10
    json.dumps(rep.to_dict())


def test_tail_energy_logged_and_decreasing():
    ksp, kern, mask, x0, rank = _small_problem()
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=4, gradient_steps=5, iterations=6)],
                             circular_axes=(0, 1), seed=7)
    _, rep = H.hicu_reconstruct(x0, mask, kern, sched)
    tails = [r.tail_energy for r in rep.iterations]
    assert all(t is not None for t in tails) and tails[-1] < tails[0]


def test_soft_mode_close_to_data():
    ksp, kern, mask, x0, rank = _small_problem()
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=3, gradient_steps=4, iterations=6)],
                             circular_axes=(0, 1), dc_mode="soft", dc_lambda=50.0, seed=8)
    xhat, _ = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    obs = mask == 1
    assert np.linalg.norm(xhat[obs] - x0[obs]) / np.linalg.norm(x0[obs]) < 0.05


def test_coil_compress_option():
    ksp, kern, mask, x0, rank = _small_problem(nc=4)
    kern3 = H.KernelMask.full((5, 5, 3))
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=3, gradient_steps=3, iterations=3)], seed=5)
    xhat, rep = H.hicu_reconstruct(x0, mask, kern3, sched, reference=ksp, tail_energy_threshold=0, coil_compress=3)
    assert xhat.shape == ksp.shape[:-1] + (3,)
    assert rep.coil_basis.shape == (4, 3)
    assert np.isfinite(rep.steps[-1].ser_db)


def test_coil_compress_fused_mask_apply():
    """The coil-compression path uploads raw k-space and applies mask_apply
    (arrays.py:54-67) on the device: unmasked garbage at unobserved points
    must give the bit-identical reconstruction of the zero-filled input.  Masks
    that differ between coils are rejected (virtual coils mix all coils)."""
    ksp, kern, mask, x0, rank = _small_problem(nc=4)
    rng = np.random.default_rng(11)
    mask = mask.copy()
    zf = np.where(mask == 1, ksp, 0).astype(np.complex64)
    junk = (ksp + 5.0 * (rng.standard_normal(ksp.shape) + 1j * rng.standard_normal(ksp.shape))).astype(np.complex64)
    raw = np.where(mask == 1, zf, junk)
    kern3 = H.KernelMask.full((5, 5, 3))
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=3, gradient_steps=3, iterations=3)], seed=5)
    a, ra = H.hicu_reconstruct(zf, mask, kern3, sched, tail_energy_threshold=0, coil_compress=3)
    b, rb = H.hicu_reconstruct(raw, mask, kern3, sched, tail_energy_threshold=0, coil_compress=3)
    assert np.array_equal(a, b)
    assert np.array_equal(ra.coil_basis, rb.coil_basis)
    per_coil = mask.copy()
    per_coil[..., 1] = (rng.random(mask.shape[:-1]) < 0.6).astype(mask.dtype)
    with pytest.raises(H.ConfigError):
        H.hicu_reconstruct(zf, per_coil, kern3, sched, tail_energy_threshold=0, coil_compress=3)


def test_gram_fp64_accuracy_3d():
    """tcgen05 and SIMT Gram against an fp64 Gram (patch matrix built by
    as_strided) on a 3-D 5x5x5x8 geometry (the C4/C5 kernels): both within
    the north star's 1e-5."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(3)
    dims, kext = (12, 40, 40, 8), (5, 5, 5, 8)
    x = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    out = tuple(s - k + 1 for s, k in zip(dims[:-1], kext[:-1]))
    st = x.stride()
    v = x.as_strided(out + kext[:-1] + (dims[-1],), st[:-1] + st[:-1] + (st[-1],)).reshape(-1, kernel.n)
    G64 = torch.zeros((kernel.n, kernel.n), dtype=torch.complex128, device="cuda")
    for i in range(0, v.shape[0], 4096):
        P = v[i:i + 4096].to(torch.complex128)
        G64 += P.conj().T @ P
    sc = float(G64.abs().max())
    for path in ("lag", "tcgen05", "simt"):  # lag (the default at n = 1000), dense tcgen05, dense SIMT
        G = H.gram_matrix(x, kernel, region, path=path)
        err = float((G - G64).abs().max()) / sc
        print(f"3-D 5x5x5x8 Gram ({path}): max rel err {err:.2e}")
        assert err <= 1e-5, path


def test_sharded_cuda_backend_single_rank():
    """The halo-sharded driver with the CUDA backend (world size 1: no
    neighbours) reproduces hicu_reconstruct on the same inputs."""
    import socket

    import torch.distributed as dist

    from paper_2004_08962_b200.parallel import sharded_reconstruct

    rng = np.random.default_rng(5)
    dims = (20, 14, 12, 8)
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    mask = np.repeat((rng.random(dims[:3] + (1,)) < 0.5).astype(np.uint8), 8, axis=3)
    x0 = np.where(mask == 1, x, 0)
    kern = H.KernelMask.full((3, 3, 3, 8))
    sched = H.SolverSchedule(rank=30, stages=[H.StageSpec("full", 4, 2, 2)], seed=2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        xs, recs = sharded_reconstruct(x0, mask, kern, sched)
    finally:
        dist.destroy_process_group()
    xr, rep = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    assert np.abs(xs - xr).max() <= 1e-5 * np.abs(xr).max()
    etas = np.concatenate(recs)[:, 3]
    assert np.allclose(etas, [st.eta for st in rep.steps], rtol=1e-4)


def test_reconstruct_slices_partition():
    from paper_2004_08962_b200.parallel import reconstruct_slices

    ksp, kern, mask, x0, rank = _small_problem()
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p=2, gradient_steps=2, iterations=1)], seed=1)
    out0 = reconstruct_slices([x0, x0, x0], [mask] * 3, kern, sched, rank=0, world=2, tail_energy_threshold=0)
    out1 = reconstruct_slices([x0, x0, x0], [mask] * 3, kern, sched, rank=1, world=2, tail_energy_threshold=0)
    assert sorted(out0) == [0, 1] and sorted(out1) == [2]
    assert np.array_equal(out0[0][0], out1[2][0])


def test_cli_recon_matches_api(tmp_path):
    """`hicu recon --config` (cli.py) writes exactly the array hicu_reconstruct
    returns and the reference's report keys (dims, rank, seed)."""
    import json as _json

    from paper_2004_08962_b200 import cli

    rng = np.random.default_rng(5)
    dims = (24, 20, 4)
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    mask = np.repeat((rng.random(dims[:2] + (1,)) < 0.5).astype(np.uint8), dims[2], axis=2)
    H.write_array(tmp_path / "k.hicu", x)
    H.write_array(tmp_path / "m.hicu", mask)
    doc = {"kernel": {"extents": [3, 3, 4]},
           "schedule": {"rank": 8, "stages": [{"region": "full", "p": 4, "gradient_steps": 2, "iterations": 3}]},
           "paths": {"kspace": "k.hicu", "mask": "m.hicu"}}
    (tmp_path / "run.json").write_text(_json.dumps(doc))
    assert cli.main(["recon", "--config", str(tmp_path / "run.json"), "--out", str(tmp_path), "--seed", "4"]) == 0
    got = H.read_array(tmp_path / "recon.hicu")
    cfg = H.parse_config(doc)
    cfg.schedule.seed = 4
    want, _ = H.hicu_reconstruct(H.mask_apply(x, mask), mask, cfg.kernel, cfg.schedule)
    assert np.array_equal(got, want)
    rep = _json.loads((tmp_path / "report.json").read_text())
    assert rep["dims"] == list(dims) and rep["rank"] == 8 and rep["seed"] == 4


REDUCED = {
    # name: (config, scale, coils kept, kernel, rank, stages) -- reduced shapes of BASELINE configs[2:5]
    "C3_slice": ("C3", 0.2, 10, (7, 7, 10), 100, [("full", 10, 5, 6)]),
    "C4_cine": ("C4", 0.25, 8, (3, 3, 3, 8), 40, [([0.5, 0.5, "full"], 8, 5, 4), ("full", 8, 5, 4)]),
    "C5_volume": ("C5", 0.15, 8, (3, 3, 3, 8), 40, [("full", 8, 5, 8)]),
    # the C5 kernel and rank (n = 1000, r = 120): streamed tcgen05 convolutions with
    # prebuilt B images and the global-memory-LU closed-form nullspace in the driver
    "C5_kernel_rank": ("C5", 0.15, 8, (5, 5, 5, 8), 120, [("full", 8, 5, 2)]),
}


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("name", list(REDUCED))
def test_reduced_config_ser_parity(name):
    """Free-running device run vs the oracle (the reference's rSVD with the
    device's canonical phase convention) on reduced shapes of C3 (10 coils,
    p = 10, 7x7 kernel: SIMT conv/Gram), C4 (3-D + time with a CO stage) and
    C5 (3-D volume): tcgen05 3-D geometries end to end."""
    from paper_2004_08962_b200.synthetic import make_config

    cfg, scale, nc, kext, rank, stages = REDUCED[name]
    ksp, mask, x0 = make_config(cfg, scale=scale)
    ksp, mask, x0 = ksp[..., :nc], mask[..., :nc], x0[..., :nc]
    kern = H.KernelMask.full(kext)
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec(*s) for s in stages], seed=0)
    xg, _ = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    xo, _ = O.hicu_reconstruct(x0, mask, kext, stages, rank, seed=0, canonical=True)
    ser_g, ser_o, ser_0 = O.ser_db(ksp, xg), O.ser_db(ksp, xo), O.ser_db(ksp, x0)
    print(f"{name} dims {x0.shape}: zero-filled {ser_0:.3f} dB, device {ser_g:.3f} dB, oracle {ser_o:.3f} dB")
    assert ser_g > ser_0
    assert abs(ser_g - ser_o) <= 0.1
    assert np.array_equal(xg[mask == 1], x0[mask == 1].astype(np.complex128))


def test_batch_concurrent_streams_bit_identical():
    """hicu_reconstruct_batch (slices on concurrent CUDA streams) returns
    exactly what sequential hicu_reconstruct calls return."""
    from paper_2004_08962_b200.synthetic import make_config

    slices = [make_config("C1", slice_index=i, scale=0.25) for i in range(3)]
    kern = H.KernelMask.full((5, 5, 8))
    sched = H.SolverSchedule(rank=20, stages=[H.StageSpec("full", 8, 3, 4)], seed=1)
    x0s = [s[2] for s in slices]
    masks = [s[1] for s in slices]
    seq = [H.hicu_reconstruct(x, m, kern, sched, tail_energy_threshold=0) for x, m in zip(x0s, masks)]
    bat = H.hicu_reconstruct_batch(x0s, masks, kern, sched, concurrency=3, tail_energy_threshold=0)
    for (xa, ra), (xb, rb) in zip(seq, bat):
        assert np.array_equal(xa, xb)
        assert [s.eta for s in ra.steps] == [s.eta for s in rb.steps]


def test_batch_cold_start_concurrent_first_launch():
    """The very first kernel launches of a process come from several host
    threads at once (hicu_reconstruct_batch); one-time launch set-up (the
    dynamic shared-memory opt-in) must not race (regression: a concurrent
    first conv_tc launch used to fail with 'invalid argument')."""
    import subprocess
    import sys

    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_2004_08962_b200 as H\n"
        "from paper_2004_08962_b200.synthetic import make_config\n"
        "sl = [make_config('C1', slice_index=i, scale=0.25) for i in range(4)]\n"
        "k = H.KernelMask.full((5, 5, 8))\n"
        "s = H.SolverSchedule(rank=20, stages=[H.StageSpec('full', 8, 2, 2)], seed=1)\n"
        "out = H.hicu_reconstruct_batch([x[2] for x in sl], [x[1] for x in sl], k, s, concurrency=4,\n"
        "                               tail_energy_threshold=0)\n"
        "print(len(out))\n"
    ) % str(ROOT)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert res.stdout.strip().endswith("4")


def _sharded_cuda_worker(rank, world, port, out_path, case):
    import os

    import torch
    import torch.distributed as dist

    from paper_2004_08962_b200.parallel import sharded_reconstruct

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x0, mask, kern, sched, axis = _sharded_case(case)
    xs, recs = sharded_reconstruct(x0, mask, kern, sched, axis=axis)
    if rank == 0:
        np.savez(out_path, xs=xs, etas=np.concatenate(recs)[:, 3])
    dist.barrier()
    dist.destroy_process_group()


def _sharded_case(case):
    rng = np.random.default_rng(9)
    if case == "readout":
        dims, kext, axis, circ = (20, 14, 12, 8), (3, 3, 3, 8), 0, ()
        stages = [H.StageSpec("full", 8, 2, 2)]
    elif case == "time_thin":  # 3 output frames over 2 ranks (2 + 1) against a 4-frame halo
        dims, kext, axis, circ = (24, 20, 7, 8), (3, 3, 5, 8), 2, ()
        stages = [H.StageSpec([16, 12, "full"], 8, 2, 1), H.StageSpec("full", 8, 2, 1)]
    else:  # circular time: a ring
        dims, kext, axis, circ = (18, 16, 9, 8), (3, 3, 5, 8), 2, (2,)
        stages = [H.StageSpec("full", 4, 2, 2)]
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    mask = np.repeat((rng.random(dims[:-1] + (1,)) < 0.5).astype(np.uint8), dims[-1], axis=len(dims) - 1)
    x0 = np.where(mask == 1, x, 0)
    sched = H.SolverSchedule(rank=30, stages=stages, circular_axes=circ, seed=2)
    return x0, mask, H.KernelMask.full(kext), sched, axis


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", ["readout", "time_thin", "time_ring"])
def test_sharded_cuda_backend_two_ranks(tmp_path, case):
    """Two processes on this GPU, gloo (host-staged halos): the CUDA backend's
    halo accumulate / refresh, the Gram and scalar all-reduces and the
    replicated nullspace reproduce the single-domain hicu_reconstruct --
    along the readout axis (C5), along time with shards thinner than the
    halo (C4), and along a circular time axis (ring)."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    path = str(tmp_path / "w2.npz")
    mp.spawn(_sharded_cuda_worker, args=(2, port, path, case), nprocs=2, join=True)
    out = np.load(path)
    x0, mask, kern, sched, axis = _sharded_case(case)
    xr, rep = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    err = np.abs(out["xs"] - xr).max() / np.abs(xr).max()
    print(f"sharded ({case}, 2 ranks) vs single domain: {err:.2e}")
    assert err <= 1e-5
    assert np.allclose(out["etas"], [st.eta for st in rep.steps], rtol=1e-4)


def _sharded_cc_worker(rank, world, port, out_path):
    import os

    import torch
    import torch.distributed as dist

    from paper_2004_08962_b200.parallel import sharded_reconstruct

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x0, mask, kern, sched = _cc_case()
    xs, _ = sharded_reconstruct(x0, mask, kern, sched, axis=2, coil_compress=4)
    if rank == 0:
        np.save(out_path, xs)
    dist.barrier()
    dist.destroy_process_group()


def _cc_case():
    from paper_2004_08962_b200.synthetic import make_config

    ksp, mask, x0 = make_config("C4", scale=0.125)  # 24 x 18 x 25 frames, 12 coils
    sched = H.SolverSchedule(rank=30, stages=[H.StageSpec([16, 12, "full"], 4, 2, 1), H.StageSpec("full", 4, 2, 1)],
                             seed=3)
    return x0, mask, H.KernelMask.full((3, 3, 5, 4)), sched


@pytest.mark.timeout(600)
def test_sharded_time_axis_coil_compression():
    """C4's pipeline at toy size, two processes: distributed SVD coil
    compression (12 -> 4: covariance all-reduced, one basis) then the
    time-sharded reconstruction, against hicu_reconstruct(coil_compress=4)."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    import tempfile

    path = tempfile.mktemp(suffix=".npy")
    mp.spawn(_sharded_cc_worker, args=(2, port, path), nprocs=2, join=True)
    xs = np.load(path)
    x0, mask, kern, sched = _cc_case()
    xr, _ = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0, coil_compress=4)
    err = np.abs(xs - xr).max() / np.abs(xr).max()
    print(f"sharded time axis + coil compression vs single domain: {err:.2e}")
    assert err <= 1e-5


def test_p32_stage_lockstep():
    """The paper's full-stage compression p = 4 Nc = 32 (the
    reference accepts any p >= 1, subspace.py:223-224): lockstep against the
    oracle with its V injected, 8 coils, 5x5x8 kernel."""
    rng = np.random.default_rng(12)
    dims = (28, 26, 8)
    img = np.zeros(dims[:2], complex)
    yy, xx = np.mgrid[:dims[0], :dims[1]] / dims[0] - 0.5
    img[(xx / 0.35) ** 2 + (yy / 0.3) ** 2 <= 1] = 1.0
    sens = np.stack([np.exp(2j * np.pi * (0.3 * k * xx - 0.2 * (k - 3) * yy)) for k in range(8)], -1)
    ksp = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(img[..., None] * sens, axes=(0, 1)), axes=(0, 1),
                                      norm="ortho"), axes=(0, 1))
    ksp = ksp + 1e-3 * np.abs(ksp).max() * (rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    mask = np.repeat((rng.random(dims[:2] + (1,)) < 0.5).astype(np.uint8), 8, axis=2)
    x0 = np.where(mask == 1, ksp, 0)
    stages = [("full", 32, 3, 2)]
    vlog, trace = {}, []
    xo, _ = O.hicu_reconstruct(x0, mask, (5, 5, 8), stages, 30, seed=1, trace=trace, v_log=vlog)
    sched = H.SolverSchedule(rank=30, stages=[H.StageSpec(*s) for s in stages], seed=1)
    xg, rep = H.hicu_reconstruct(x0, mask, H.KernelMask.full((5, 5, 8)), sched, tail_energy_threshold=0,
                                 lockstep_v=lambda si, it: vlog[(si, it)])
    eo = np.array([t["eta"] for t in trace])
    eg = np.array([s.eta for s in rep.steps])
    assert np.abs(eg - eo).max() <= 1e-4 * np.abs(eo).max()
    assert np.linalg.norm(xg - xo) <= 1e-5 * np.linalg.norm(xo)


def test_native_nccl_collectives_single_rank():
    """The library's NCCL communicator (hicu_comm_*, hicu_allreduce,
    hicu_halo_exchange) at world size 1: the all-reduce is the identity, a
    grouped self send/receive copies the buffer, and the sharded driver on
    the native communicator reproduces hicu_reconstruct."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2004_08962_b200 import _native as nat
    from paper_2004_08962_b200.parallel import NativeComm, sharded_reconstruct

    assert nat.lib().hicu_comm_available()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = NativeComm()
        t = torch.arange(10, dtype=torch.float64, device="cuda")
        comm.allreduce_(t)
        src = torch.randn(1000, device="cuda")
        dst = torch.zeros_like(src)
        comm.exchange([(0, nat.P2P_SEND, src), (0, nat.P2P_RECV, dst)])
        torch.cuda.synchronize()
        assert torch.equal(t, torch.arange(10, dtype=torch.float64, device="cuda"))
        assert torch.equal(src, dst)
        comm.close()
        x0, mask, kern, sched, axis = _sharded_case("time_ring")  # a ring onto itself
        xs, recs = sharded_reconstruct(x0, mask, kern, sched, axis=axis, native_comm=True)
    finally:
        dist.destroy_process_group()
    xr, rep = H.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
    assert np.abs(xs - xr).max() <= 1e-5 * np.abs(xr).max()
