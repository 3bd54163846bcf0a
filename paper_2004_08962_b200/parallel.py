"""Multi-GPU execution of the HICU path.

Two modes, one process per GPU (torchrun), ``torch.distributed`` for the
plumbing:

* **Independent slices (C3)** — :func:`partition_slices` /
  :func:`reconstruct_slices`: every rank reconstructs its own contiguous block
  of slices; there is no data-path collective (weak scaling).

* **One volume sharded along axis 0 (C5)** — :class:`ShardPlan` /
  :class:`ShardedReconstruction`: the region's output rows on axis 0 are
  split into contiguous blocks; rank k owns k-space planes [P_k, P_{k+1}) and
  holds K0-1 trailing halo planes.  Per outer iteration the local Gram
  partials are all-reduced (n x n complex128) and the nullspace step runs
  redundantly (bit-identical on every rank).  Per gradient step:
    conv_fwd (local rows) -> raw scatter over local planes
    -> halo ACCUMULATE: trailing partial g -> next rank, added to its first
       K0-1 owned planes
    -> data consistency on owned planes
    -> halo REFRESH: first K0-1 owned planes of g -> previous rank's halo
    -> ELS conv (local rows) -> all-reduce of 7 scalar sums -> the same eta
       everywhere -> y -= eta g on owned AND halo planes (the halo update is
       bit-identical to the owner's, so y never needs an exchange).
  Flops are partitioned exactly by output row; only the halos are replicated.

The compute backend is pluggable: :class:`CudaShardBackend` drives
``libhicu_b200.so``; tests drive the same host logic with a CPU backend and
the ``gloo`` process group (world size 2) to check it against a single
domain.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

__all__ = [
    "partition_slices",
    "reconstruct_slices",
    "ShardPlan",
    "HaloExchange",
    "ShardedReconstruction",
    "CudaShardBackend",
]


def partition_slices(n_slices: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of slice indices for ``rank`` (first
    ``n_slices % world`` ranks get one extra)."""
    if world < 1 or not (0 <= rank < world):
        raise ConfigError("invalid world/rank")
    base, extra = divmod(int(n_slices), int(world))
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def reconstruct_slices(x0_slices, masks, kernel, schedule, rank: int = 0, world: int = 1, concurrency: int = 4,
                       **kw):
    """C3-style slice parallelism: reconstruct this rank's block of
    independent slices, ``concurrency`` at a time on separate CUDA streams
    (:func:`hicu_reconstruct_batch`); returns ``{slice_index: (xhat, report)}``.
    No collective on the data path."""
    from .solver import hicu_reconstruct_batch

    idx = list(partition_slices(len(x0_slices), world, rank))
    res = hicu_reconstruct_batch([x0_slices[s] for s in idx], [masks[s] for s in idx], kernel, schedule,
                                 concurrency=concurrency, **kw)
    return dict(zip(idx, res))


def split_rows(n_rows: int, world: int):
    """Balanced contiguous blocks of [0, n_rows): list of (r0, r1)."""
    return [(r.start, r.stop) for r in (partition_slices(n_rows, world, k) for k in range(world))]


@dataclass
class ShardPlan:
    """Plane ownership for a volume sharded along axis 0.

    ``rows`` are the region's output rows on axis 0 (offset ``roff``); rank k
    owns k-space planes [P[k], P[k+1]) and holds planes
    [P[k], min(D, P[k+1] + K0 - 1)) locally."""

    dims: tuple
    k0: int
    roff: int
    rext: int
    world: int
    rank: int

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        D = self.dims[0]
        blocks = split_rows(self.rext, self.world)
        self.rows = blocks
        self.P = [0] + [self.roff + b[0] for b in blocks[1:]] + [D]
        halo = self.k0 - 1
        for k in range(self.world):
            if self.P[k + 1] - self.P[k] < max(halo, 1):
                raise ConfigError(f"shard {k} owns {self.P[k + 1] - self.P[k]} planes, fewer than the "
                                  f"{halo}-plane halo; use fewer ranks")
        self.halo = halo

    @property
    def r0(self) -> int:
        return self.rows[self.rank][0]

    @property
    def r1(self) -> int:
        return self.rows[self.rank][1]

    @property
    def plane_lo(self) -> int:
        return self.P[self.rank]

    @property
    def plane_hi(self) -> int:
        """One past the last locally held plane (owned + trailing halo)."""
        return min(self.dims[0], self.P[self.rank + 1] + self.halo)

    @property
    def owned(self) -> int:
        return self.P[self.rank + 1] - self.P[self.rank]

    @property
    def local_dims(self) -> tuple:
        return (self.plane_hi - self.plane_lo,) + self.dims[1:]

    @property
    def local_roff0(self) -> int:
        return self.roff + self.r0 - self.plane_lo

    @property
    def trailing(self) -> int:
        """Halo planes held after the owned block."""
        return self.plane_hi - self.P[self.rank + 1]


class HaloExchange:
    """Neighbour exchanges of plane blocks over ``torch.distributed`` (NCCL for
    CUDA tensors, gloo for CPU tensors).  Tensors are (planes, ...) with
    axis 0 the sharded axis, contiguous."""

    def __init__(self, plan: ShardPlan, group=None):
        import torch.distributed as dist

        self.plan = plan
        self.group = group
        self.dist = dist

    def _exchange(self, send_to, send_buf, recv_from, recv_buf):
        dist = self.dist
        ops = []
        if send_to is not None:
            ops.append(dist.P2POp(dist.isend, send_buf.contiguous(), send_to, group=self.group))
        if recv_from is not None:
            ops.append(dist.P2POp(dist.irecv, recv_buf, recv_from, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def accumulate(self, g_local):
        """Send my trailing halo partials to the next rank; add the previous
        rank's trailing partials into my first owned planes."""
        import torch

        pl = self.plan
        nxt = pl.rank + 1 if pl.rank + 1 < pl.world else None
        prv = pl.rank - 1 if pl.rank > 0 else None
        send = g_local[pl.owned:pl.owned + pl.trailing] if nxt is not None else None
        recv = None
        if prv is not None:
            prev_plan = ShardPlan(pl.dims, pl.k0, pl.roff, pl.rext, pl.world, prv)
            recv = torch.empty((prev_plan.trailing,) + tuple(g_local.shape[1:]), dtype=g_local.dtype,
                               device=g_local.device)
        self._exchange(nxt, send, prv, recv)
        if recv is not None:
            g_local[:recv.shape[0]] += recv

    def refresh(self, g_local):
        """Send my first owned planes to the previous rank's halo; receive my
        trailing halo from the next rank."""
        pl = self.plan
        nxt = pl.rank + 1 if pl.rank + 1 < pl.world else None
        prv = pl.rank - 1 if pl.rank > 0 else None
        send = None
        if prv is not None:
            prev_plan = ShardPlan(pl.dims, pl.k0, pl.roff, pl.rext, pl.world, prv)
            send = g_local[:prev_plan.trailing]
        recv = g_local[pl.owned:pl.owned + pl.trailing] if nxt is not None else None
        if recv is not None and not recv.is_contiguous():
            raise ConfigError("halo block must be contiguous")
        self._exchange(prv, send, nxt, recv)

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t


class ShardedReconstruction:
    """The solver loop (solver.py:322-393) on one axis-0 shard of a volume.

    ``backend`` provides the local compute (see :class:`CudaShardBackend`);
    all ranks must pass identical ``x0/mask/kernel/schedule``."""

    def __init__(self, backend, plan: ShardPlan, halo: HaloExchange):
        self.b = backend
        self.plan = plan
        self.halo = halo

    def run_iteration(self, si: int, it: int):
        """One outer iteration of stage ``si`` (the unit a benchmark step
        times): Gram partials -> all-reduce -> redundant nullspace -> G
        gradient steps with their halo exchanges and scalar all-reduces."""
        b, pl, hx = self.b, self.plan, self.halo
        stage = b.schedule.stages[si]
        G = b.gram(si)
        hx.allreduce_(b.as_real(G))
        b.nullspace(si, it, G)
        for j in range(stage.gradient_steps):
            b.conv_fwd(si, j)
            g = b.scatter_raw(si, j)
            hx.accumulate(g)
            b.dc_apply(pl.owned)
            hx.refresh(g)
            b.conv_els(si, j)
            sums = b.reduce()
            hx.allreduce_(sums)
            b.apply(si, it, j, sums)

    def run(self):
        for si, stage in enumerate(self.b.schedule.stages):
            for it in range(stage.iterations):
                self.run_iteration(si, it)
        return self.b.result()


def plan_for(dims, kernel, schedule, world: int, rank: int) -> ShardPlan:
    """Shard plan along axis 0; every stage must span axis 0 in full."""
    from .solver import stage_region

    regs = [stage_region(dims, kernel, st.region, schedule.circular_axes) for st in schedule.stages]
    if 0 in set(schedule.circular_axes):
        raise ConfigError("axis 0 must not be circular in sharded mode")
    r0 = {(r.offsets[0], r.extents[0]) for r in regs}
    if len(r0) != 1:
        raise ConfigError("sharded mode needs the same axis-0 region in every stage")
    roff, rext = r0.pop()
    return ShardPlan(tuple(dims), kernel.extents[0], roff, rext, world, rank)


class CudaShardBackend:
    """Local compute of one shard on the current CUDA device through the C ABI."""

    def __init__(self, x0, mask, kernel, schedule, plan: ShardPlan):
        from . import _native as nat
        from .hankel import Region, device_geometry, to_dev
        from .solver import ReconEngine, draw_stage, stage_region

        self.nat = nat
        self.torch = nat.require_cuda()
        torch = self.torch
        self.schedule = schedule
        self.plan = plan
        self.kernel = kernel
        lo, hi = plan.plane_lo, plan.plane_hi
        x0 = np.asarray(x0)
        mask = np.asarray(mask)
        observed = mask == 1
        xm = np.where(observed, x0, 0).astype(np.complex64)[lo:hi]
        self.mask_np = observed.astype(np.uint8)[lo:hi]
        ldims = plan.local_dims
        self.regions = []
        for st in schedule.stages:
            rg = stage_region(x0.shape, kernel, st.region, schedule.circular_axes)
            offs = (plan.local_roff0,) + rg.offsets[1:]
            exts = (plan.r1 - plan.r0,) + rg.extents[1:]
            self.regions.append(Region(offs, exts, rg.circular_axes))
        self.eng = ReconEngine(xm, self.mask_np, ldims, kernel, schedule, self.regions)
        for si, st in enumerate(schedule.stages):
            om, pb = draw_stage(schedule, si, st, kernel.n)
            self.eng.set_host_draws(si, om, pb)
        self.geoms = [device_geometry(kernel, rg, ldims) for rg in self.regions]
        self.sums = torch.zeros(8, dtype=torch.float64, device="cuda")
        e = self.eng
        self.dc_parts = torch.zeros(4 * nat.lib().hicu_dc_nparts(max(1, plan.owned * int(np.prod(ldims[1:])))),
                                    dtype=torch.float64, device="cuda")
        self.plane = int(np.prod(ldims[1:]))
        self.ldims = ldims

    @staticmethod
    def as_real(G):
        return G.view(G.real.dtype) if G.is_complex() else G

    def _st(self):
        return self.nat.stream_handle()

    def gram(self, si):
        e, L = self.eng, self.nat.lib()
        self.nat.check(L.hicu_gram(self.geoms[si].ref(), e.y.data_ptr(), e.G.data_ptr(), e.gram_ws.data_ptr(),
                                   e.gram_bytes, self._st()), "gram")
        return e.G

    def nullspace(self, si, it, G):
        e, L, nat = self.eng, self.nat.lib(), self.nat
        n, r, ell = e.n, e.r, e.ell
        st = self.schedule.stages[si]
        om, pb = e.stage_data[si]
        nat.check(L.hicu_nystrom(n, ell, r, G.data_ptr(), om[it].data_ptr(), e.V.data_ptr(), e.nys_ws.data_ptr(),
                                 e.nys_bytes, e.status.data_ptr(), self._st()), "nystrom")
        nat.check(L.hicu_householder(n, r, e.V.data_ptr(), 1e-12, e.refl.data_ptr(), e.tau.data_ptr(),
                                     e.flags.data_ptr(), e.status.data_ptr(), self._st()), "householder")
        nat.check(L.hicu_apply_reflectors(n, r, e.refl.data_ptr(), e.tau.data_ptr(), e.flags.data_ptr(),
                                          st.gradient_steps * st.p, pb[it].data_ptr(), e.B.data_ptr(),
                                          e.qt32.data_ptr(), st.p, self._st()), "reflectors")

    def _qt(self, si, j):
        e = self.eng
        st = self.schedule.stages[si]
        return e.qt32.data_ptr() + j * e.n * st.p * 8

    def conv_fwd(self, si, j):
        e, L = self.eng, self.nat.lib()
        self._si = si
        self.nat.check(L.hicu_conv_fwd(self.geoms[si].ref(), e.y.data_ptr(), self._qt(si, j),
                                       self.schedule.stages[si].p, e.u.data_ptr(), e.obj_parts.data_ptr(),
                                       self._st()), "conv_fwd")

    def scatter_raw(self, si, j):
        e, L = self.eng, self.nat.lib()
        self.nat.check(L.hicu_scatter_dc(self.geoms[si].ref(), self._qt(si, j), self.schedule.stages[si].p,
                                         e.u.data_ptr(), e.mask.data_ptr(), None, None, 2, 0.0, e.g.data_ptr(),
                                         e.dc_parts.data_ptr(), self._st()), "scatter")
        return e.g.view(self.ldims[0], -1)

    def dc_apply(self, owned_planes):
        e, L = self.eng, self.nat.lib()
        n = owned_planes * self.plane
        soft = self.schedule.dc_mode == "soft"
        self.nat.check(L.hicu_dc_apply(n, e.g.data_ptr(), e.mask.data_ptr(), e.y.data_ptr(),
                                       e.x0.data_ptr() if soft else None, 1 if soft else 0,
                                       float(self.schedule.dc_lambda) if soft else 0.0, self.dc_parts.data_ptr(),
                                       self._st()), "dc_apply")
        self._ndc = self.nat.lib().hicu_dc_nparts(n)

    def conv_els(self, si, j):
        e, L = self.eng, self.nat.lib()
        self.nat.check(L.hicu_conv_els(self.geoms[si].ref(), e.g.data_ptr(), self._qt(si, j),
                                       self.schedule.stages[si].p, e.u.data_ptr(), e.els_parts.data_ptr(),
                                       self._st()), "conv_els")

    def reduce(self):
        e, L = self.eng, self.nat.lib()
        ncp = self.geoms[self._si].conv_nparts
        self.nat.check(L.hicu_step_reduce(e.obj_parts.data_ptr(), ncp, self.dc_parts.data_ptr(), self._ndc,
                                          e.els_parts.data_ptr(), ncp, self.sums.data_ptr(), self._st()), "reduce")
        return self.sums

    def apply(self, si, it, j, sums):
        e, L = self.eng, self.nat.lib()
        st = self.schedule.stages[si]
        rec = e.recs[si].data_ptr() + (it * st.gradient_steps + j) * self.nat.REC_SLOTS * 8
        soft = self.schedule.dc_mode == "soft"
        self.nat.check(L.hicu_step_apply(e.N, e.y.data_ptr(), e.g.data_ptr(), sums.data_ptr(), 1 if soft else 0,
                                         float(self.schedule.dc_lambda) if soft else 0.0, rec, self._st()),
                       "apply")

    def result(self):
        """(owned planes of y as complex128, per-stage record arrays)."""
        pl = self.plan
        y = self.eng.y.view(self.ldims)[:pl.owned].cpu().numpy().astype(np.complex128)
        recs = [r.cpu().numpy().reshape(-1, self.nat.REC_SLOTS) for r in self.eng.recs]
        return y, recs


def gather_planes(local_owned, plan: ShardPlan, group=None):
    """All-gather the owned planes of every rank into the full volume
    (rank order = plane order).  Works for CPU (gloo) and CUDA (NCCL)."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(local_owned)
    maxp = max(plan.P[k + 1] - plan.P[k] for k in range(plan.world))
    pad = torch.zeros((maxp,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    if pad.is_complex():
        pad_r = torch.view_as_real(pad).contiguous()
    else:
        pad_r = pad
    outs = [torch.empty_like(pad_r) for _ in range(plan.world)]
    dist.all_gather(outs, pad_r, group=group)
    blocks = []
    for k in range(plan.world):
        o = torch.view_as_complex(outs[k]) if pad.is_complex() else outs[k]
        blocks.append(o[:plan.P[k + 1] - plan.P[k]])
    return torch.cat(blocks, dim=0)


def sharded_reconstruct(x0, mask, kernel, schedule, group=None):
    """Reconstruct one volume sharded along axis 0 over the ranks of
    ``group`` (one GPU per rank).  Returns (xhat complex128 full volume,
    records of this rank's run: list per stage of [iters*G, 8] arrays)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = plan_for(np.asarray(x0).shape, kernel, schedule, world, rank)
    backend = CudaShardBackend(x0, mask, kernel, schedule, plan)
    halo = HaloExchange(plan, group)
    y_owned, recs = ShardedReconstruction(backend, plan, halo).run()
    import torch

    full = gather_planes(torch.from_numpy(y_owned).cuda(), plan, group).cpu().numpy()
    obs = np.asarray(mask) == 1
    if schedule.dc_mode == "hard":
        full[obs] = np.asarray(x0, np.complex128)[obs]
    return full, recs
