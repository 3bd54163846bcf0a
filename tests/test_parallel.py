"""Multi-rank host logic on the CPU with the gloo backend.

The sharded driver (plane ownership, halo accumulate/refresh, Gram and
scalar all-reduces) is exercised with a CPU compute backend built from the
oracle, world size 2, and must reproduce the single-domain run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2004_08962_b200 as H
from paper_2004_08962_b200.parallel import (HaloExchange, ShardPlan, ShardedReconstruction, gather_planes,
                                            partition_slices, plan_for, split_rows)
from paper_2004_08962_b200.solver import draw_stage, stage_region
from oracle import hicu_oracle as O


def test_partition_slices_balanced():
    for n, w in [(64, 8), (64, 3), (5, 8), (7, 2)]:
        blocks = [partition_slices(n, w, r) for r in range(w)]
        flat = [i for b in blocks for i in b]
        assert flat == list(range(n))
        sizes = [len(b) for b in blocks]
        assert max(sizes) - min(sizes) <= 1


def test_shard_plan_planes():
    pl = [ShardPlan((256, 160, 160, 8), 5, 0, 252, 8, k) for k in range(8)]
    assert [p.r1 - p.r0 for p in pl] == [32, 32, 32, 32, 31, 31, 31, 31]
    # owned planes tile [0, D); every rank holds K0-1 trailing halo planes except the last
    assert pl[0].plane_lo == 0 and pl[-1].P[-1] == 256
    assert sum(p.owned for p in pl) == 256
    assert all(p.trailing == 4 for p in pl[:-1]) and pl[-1].trailing == 0
    with pytest.raises(H.ConfigError):
        ShardPlan((20, 8, 2), 5, 0, 6, 8, 0)  # more ranks than output rows


def test_shard_plan_time_axis_thin_shards():
    """C4: 21 valid output frames over 8 GPUs (3,3,3,3,3,2,2,2) against a
    4-frame halo: trailing halos span two neighbours; circular time: a ring."""
    dims = (192, 144, 25, 8)
    pl = [ShardPlan(dims, 5, 0, 21, 8, k, axis=2) for k in range(8)]
    assert [p.r1 - p.r0 for p in pl] == [3, 3, 3, 3, 3, 2, 2, 2]
    assert sum(p.owned for p in pl) == 25 and pl[-1].owned == 6  # the last rank also owns the 4 tail frames
    assert pl[5].planes == [15, 16, 17, 18, 19, 20] and pl[5].local_dims == (192, 144, 6, 8)
    # rank 5 (planes 15-16) reads frames 17-20: two from rank 6, two from rank 7
    assert pl[5].trailing_runs() == [(2, 2, 6, 0), (4, 2, 7, 0)]
    ring = [ShardPlan(dims, 5, 0, 25, 8, k, axis=2, circular=True) for k in range(8)]
    assert [p.owned for p in ring] == [4, 3, 3, 3, 3, 3, 3, 3]
    assert ring[7].planes == [22, 23, 24, 0, 1, 2, 3]            # wraps onto ranks 0 (and 1)
    assert ring[7].trailing_runs() == [(3, 4, 0, 0)]
    assert ring[6].trailing_runs() == [(3, 3, 7, 0), (6, 1, 0, 0)]


class CpuBackend:
    """Oracle-based local compute (complex128, torch CPU tensors)."""

    def __init__(self, x0, mask, kext, schedule, plan):
        self.schedule = schedule
        self.plan = plan
        ax = plan.axis
        obs = mask == 1
        self.y = torch.from_numpy(np.take(np.where(obs, x0, 0).astype(np.complex128), plan.planes, axis=ax).copy())
        self.x0 = self.y.clone()
        self.mask = torch.from_numpy(np.take(obs, plan.planes, axis=ax).copy())
        self.ldims = tuple(self.y.shape)
        self.kext = kext
        kern = H.KernelMask.full(kext)
        self.geoms = []
        for st in schedule.stages:
            rg = stage_region(x0.shape, kern, st.region, schedule.circular_axes)
            offs, exts = list(rg.offsets), list(rg.extents)
            offs[ax], exts[ax] = plan.local_roff0, plan.r1 - plan.r0
            circ = frozenset(a for a in rg.circular_axes if a != ax)
            self.geoms.append(O.Geom(self.ldims, kern.positions, tuple(offs), tuple(exts), circ))
        self.draws = [draw_stage(schedule, si, st, kern.n) for si, st in enumerate(schedule.stages)]
        self.recs = [np.zeros((st.iterations * st.gradient_steps, 8)) for st in schedule.stages]

    @staticmethod
    def as_real(G):
        return torch.view_as_real(G)

    def gram(self, si):
        self.G = torch.from_numpy(O.gram(self.y.numpy(), self.geoms[si]))
        return self.G

    def nullspace(self, si, it, G):
        r = self.schedule.rank
        om, pb = self.draws[si]
        v = O.canonicalize_phases(O.nystrom_right_vectors(G.numpy(), om[it], r))
        q = O.householder_nullspace(v)
        p, gs = self.schedule.stages[si].p, self.schedule.stages[si].gradient_steps
        self.qt = [q @ pb[it][r:, j * p:(j + 1) * p] for j in range(gs)]

    def conv_fwd(self, si, j):
        self.si, self.j = si, j
        self.u = O.hankel_apply(self.y.numpy(), self.qt[j], self.geoms[si])
        self.obj = float(np.vdot(self.u, self.u).real)

    def scatter_raw(self, si, j):
        self.g = torch.from_numpy(O.kspace_adjoint_scatter(self.qt[j], self.u, self.geoms[si]))
        return self.g

    def dc_apply(self, owned):
        ax = self.plan.axis
        g, m, y, x0 = (t.narrow(ax, 0, owned) for t in (self.g, self.mask, self.y, self.x0))
        lam = self.schedule.dc_lambda
        if self.schedule.dc_mode == "hard":
            g[m] = 0
            self.dc = [float((g.abs() ** 2).sum()), 0.0, 0.0, 0.0]
        else:
            res = torch.where(m, y - x0, torch.zeros_like(y))
            g += lam * res
            mg = torch.where(m, g, torch.zeros_like(g))
            self.dc = [float((g.abs() ** 2).sum()), float((res.abs() ** 2).sum()),
                       float((mg.conj() * res).sum().real), float((mg.abs() ** 2).sum())]

    def conv_els(self, si, j):
        w = O.hankel_apply(self.g.numpy(), self.qt[j], self.geoms[si])
        self.num = float(np.vdot(w, self.u).real)
        self.den = float(np.vdot(w, w).real)

    def reduce(self):
        return torch.tensor([self.obj, *self.dc, self.num, self.den, 0.0], dtype=torch.float64)

    def apply(self, si, it, j, s):
        s = s.numpy()
        lam = self.schedule.dc_lambda if self.schedule.dc_mode == "soft" else 0.0
        obj, num, den = s[0] + lam * s[2], s[5] + lam * s[3], s[6] + lam * s[4]
        eta = num / den if den > 0 else 0.0
        if den > 0:
            self.y -= eta * self.g
        self.recs[si][it * self.schedule.stages[si].gradient_steps + j, :4] = [obj, num, den, eta]

    def result(self):
        return self.y.narrow(self.plan.axis, 0, self.plan.owned).numpy(), self.recs


def _problem():
    rng = np.random.default_rng(3)
    dims = (16, 10, 9, 2)
    base = rng.standard_normal((5, 2)) + 1j * rng.standard_normal((5, 2))
    grid = np.stack(np.meshgrid(*[np.arange(d) for d in dims[:3]], indexing="ij"), -1)
    x = np.zeros(dims, complex)
    for t in range(5):  # a few separable exponentials: low-rank lifted matrix
        f = rng.uniform(0, 2 * np.pi, 3)
        x += np.exp(1j * (grid @ f))[..., None] * base[t]
    x += 0.01 * (rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    mask = np.repeat((rng.random(dims[:3] + (1,)) < 0.5).astype(np.uint8), 2, axis=3)
    x0 = np.where(mask == 1, x, 0)
    sched = H.SolverSchedule(rank=12, stages=[H.StageSpec("full", 3, 2, 2), H.StageSpec([1.0, 0.8, 0.8], 2, 2, 1)],
                             seed=4)
    return x0, mask, (3, 3, 3, 2), sched


def _worker(rank, world, port, out_path, dc_mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x0, mask, kext, sched = _problem()
    sched.dc_mode = dc_mode
    sched.dc_lambda = 2.0 if dc_mode == "soft" else 0.0
    plan = plan_for(x0.shape, H.KernelMask.full(kext), sched, world, rank)
    b = CpuBackend(x0, mask, kext, sched, plan)
    y, recs = ShardedReconstruction(b, plan, HaloExchange(plan)).run()
    full = gather_planes(torch.from_numpy(y), plan).numpy()
    if rank == 0:
        np.savez(out_path, full=full, recs=np.concatenate(recs))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dc_mode", ["hard", "soft"])
def test_sharded_two_ranks_match_single_domain(tmp_path, dc_mode):
    outs = {}
    for world in (1, 2):
        path = str(tmp_path / f"w{world}.npz")
        mp.spawn(_worker, args=(world, _free_port(), path, dc_mode), nprocs=world, join=True)
        outs[world] = np.load(path)
    a, b = outs[1], outs[2]
    assert np.allclose(a["recs"], b["recs"], rtol=1e-9, atol=1e-12)
    assert np.abs(a["full"] - b["full"]).max() <= 1e-9 * np.abs(a["full"]).max()
    # and the single-domain run is the oracle's own algorithm (Gram+Nystrom, canonical phases)
    x0, mask, kext, sched = _problem()
    xo, _ = O.hicu_reconstruct(x0, mask, kext, [(s.region, s.p, s.gradient_steps, s.iterations)
                                                for s in sched.stages], sched.rank, seed=sched.seed,
                               nullspace="nystrom", canonical=True, dc_mode=dc_mode,
                               dc_lambda=2.0 if dc_mode == "soft" else 0.0)
    xs = np.where(mask == 1, x0, a["full"]) if dc_mode == "hard" else a["full"]
    assert np.abs(xs - xo).max() <= 1e-9 * np.abs(xo).max()


def _problem_t(circular):
    """2D+t series (C4's structure at toy size): 9 frames, a 3x3x5x2 kernel
    (4-frame halo), center-out x/y window then the full grid."""
    rng = np.random.default_rng(8)
    dims = (10, 8, 9, 2)
    base = rng.standard_normal((4, 2)) + 1j * rng.standard_normal((4, 2))
    grid = np.stack(np.meshgrid(*[np.arange(d) for d in dims[:3]], indexing="ij"), -1)
    x = np.zeros(dims, complex)
    for t in range(4):
        f = rng.uniform(0, 2 * np.pi, 3)
        f[2] = 2 * np.pi * rng.integers(0, 9) / 9  # periodic in time (the cine ring)
        x += np.exp(1j * (grid @ f))[..., None] * base[t]
    x += 0.01 * (rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    mask = np.repeat((rng.random(dims[:3] + (1,)) < 0.5).astype(np.uint8), 2, axis=3)
    x0 = np.where(mask == 1, x, 0)
    sched = H.SolverSchedule(rank=10, stages=[H.StageSpec([8, 6, "full"], 2, 2, 1), H.StageSpec("full", 3, 2, 2)],
                             circular_axes=(2,) if circular else (), seed=6)
    return x0, mask, (3, 3, 5, 2), sched


def _worker_t(rank, world, port, out_path, circular):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x0, mask, kext, sched = _problem_t(circular)
    plan = plan_for(x0.shape, H.KernelMask.full(kext), sched, world, rank, axis=2)
    b = CpuBackend(x0, mask, kext, sched, plan)
    y, recs = ShardedReconstruction(b, plan, HaloExchange(plan)).run()
    full = gather_planes(torch.from_numpy(y), plan).numpy()
    if rank == 0:
        np.savez(out_path, full=full, recs=np.concatenate(recs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("circular", [False, True])
def test_time_sharded_multi_neighbour_halo(tmp_path, circular):
    """C4-style time sharding with shards thinner than the halo (world 4:
    1-2 frames per rank against a 4-frame halo) and, circularly, a ring:
    world 2 and 4 reproduce the single domain to 1e-9."""
    outs = {}
    for world in (1, 2, 4):
        path = str(tmp_path / f"t{world}.npz")
        mp.spawn(_worker_t, args=(world, _free_port(), path, circular), nprocs=world, join=True)
        outs[world] = np.load(path)
    a = outs[1]
    for world in (2, 4):
        b = outs[world]
        assert np.allclose(a["recs"], b["recs"], rtol=1e-9, atol=1e-12), world
        assert np.abs(a["full"] - b["full"]).max() <= 1e-9 * np.abs(a["full"]).max(), world
    # the single-domain run is the oracle's algorithm (Gram+Nystrom, canonical phases)
    x0, mask, kext, sched = _problem_t(circular)
    xo, _ = O.hicu_reconstruct(x0, mask, kext, [(s.region, s.p, s.gradient_steps, s.iterations)
                                                for s in sched.stages], sched.rank, seed=sched.seed,
                               circular=sched.circular_axes, nullspace="nystrom", canonical=True)
    xs = np.where(mask == 1, x0, a["full"])
    assert np.abs(xs - xo).max() <= 1e-9 * np.abs(xo).max()
