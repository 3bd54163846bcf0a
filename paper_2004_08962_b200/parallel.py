"""Multi-GPU execution of the HICU path.

Two modes, one process per GPU (torchrun), ``torch.distributed`` for the
plumbing:

* **Independent slices (C3)** — :func:`partition_slices` /
  :func:`reconstruct_slices`: every rank reconstructs its own contiguous block
  of slices; there is no data-path collective (weak scaling).

* **One volume sharded along one axis (C5: readout; C4: time)** —
  :class:`ShardPlan` / :class:`ShardedReconstruction`: the region's output
  rows on that axis are split into contiguous blocks; rank k owns k-space
  planes [P_k, P_{k+1}) and holds the K-1 trailing halo planes its rows read
  (spanning several neighbours when a shard is thinner than the halo, and
  wrapping around as a ring on a circular axis).  Per outer iteration the local Gram
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
    "NativeComm",
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


def reconstruct_slices(x0_slices, masks, kernel, schedule, rank: int = 0, world: int = 1, concurrency: int = 8,
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
    """Plane ownership for a volume sharded along one axis (``axis``).

    ``rows`` are the region's output rows on that axis (offset ``roff``); rank
    k owns k-space planes [P[k], P[k+1]) and holds, after them, the K-1
    trailing halo planes its output rows read (K = the kernel extent on the
    axis).  A shard may be thinner than its halo (C4: 21 output frames over 8
    GPUs against a 4-frame halo): the trailing halo then spans several
    neighbours.  On a circular axis (``circular``, region = the whole axis)
    the planes wrap: the last rank's halo is the first ranks' planes (a ring)."""

    dims: tuple
    k0: int
    roff: int
    rext: int
    world: int
    rank: int
    axis: int = 0
    circular: bool = False

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        D = self.dims[self.axis]
        if self.rext < self.world:
            raise ConfigError(f"{self.rext} output rows on axis {self.axis} cannot be shared by {self.world} ranks")
        blocks = split_rows(self.rext, self.world)
        self.rows = blocks
        if self.circular:
            if self.roff != 0 or self.rext != D:
                raise ConfigError("a circular sharded axis must carry the full region")
            self.P = [b[0] for b in blocks] + [D]
        else:
            self.P = [0] + [self.roff + b[0] for b in blocks[1:]] + [D]
        self.halo = self.k0 - 1
        for k in range(self.world):
            if self.P[k + 1] - self.P[k] < 1:
                raise ConfigError(f"shard {k} owns no plane; use fewer ranks")

    def for_rank(self, k: int) -> "ShardPlan":
        return ShardPlan(self.dims, self.k0, self.roff, self.rext, self.world, k, self.axis, self.circular)

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
        """One past the last locally held plane (owned + trailing halo; may
        exceed the axis length on a circular axis)."""
        if self.circular:
            return self.P[self.rank + 1] + self.halo
        return min(self.dims[self.axis], self.P[self.rank + 1] + self.halo)

    @property
    def owned(self) -> int:
        return self.P[self.rank + 1] - self.P[self.rank]

    @property
    def planes(self) -> list:
        """Global plane index of every local plane (owned, then halo)."""
        D = self.dims[self.axis]
        return [p % D for p in range(self.plane_lo, self.plane_hi)]

    @property
    def local_dims(self) -> tuple:
        d = list(self.dims)
        d[self.axis] = self.plane_hi - self.plane_lo
        return tuple(d)

    @property
    def local_roff0(self) -> int:
        return 0 if self.circular else self.roff + self.r0 - self.plane_lo

    @property
    def trailing(self) -> int:
        """Halo planes held after the owned block."""
        return self.plane_hi - self.P[self.rank + 1]

    def owner(self, p: int) -> int:
        p %= self.dims[self.axis]
        for k in range(self.world):
            if self.P[k] <= p < self.P[k + 1]:
                return k
        raise ValueError(p)

    def trailing_runs(self):
        """Runs of trailing halo planes with one owner: (local start, count,
        owner, start in the owner's local planes)."""
        runs = []
        pl = self.planes
        for i in range(self.owned, len(pl)):
            o = self.owner(pl[i])
            oi = pl[i] - self.P[o]
            if runs and runs[-1][2] == o and runs[-1][0] + runs[-1][1] == i and runs[-1][3] + runs[-1][1] == oi:
                runs[-1][1] += 1
            else:
                runs.append([i, 1, o, oi])
        return [tuple(r) for r in runs]


class NativeComm:
    """The library's own NCCL communicator (hicu_comm_*) over the ranks of a
    ``torch.distributed`` group: the unique id is made on the group's rank 0
    and broadcast by the host; collectives then run from C on the compute
    stream (hicu_allreduce, hicu_halo_exchange) without torch in the loop."""

    def __init__(self, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _native as nat

        self.nat = nat
        L = nat.lib()
        if not L.hicu_comm_available():
            raise RuntimeError("libnccl.so.2 is not loadable")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        idbuf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            nat.check(L.hicu_comm_unique_id(idbuf), "comm_unique_id")
        obj = [bytes(idbuf.raw)]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        idbuf = ctypes.create_string_buffer(obj[0], 128)
        self.h = ctypes.c_void_p()
        nat.check(L.hicu_comm_init(self.world, self.rank, idbuf, ctypes.byref(self.h)), "comm_init")

    def allreduce_(self, t):
        """In-place sum of a float64 (or complex128, as float64 pairs) device tensor."""
        v = t.view(t.real.dtype) if t.is_complex() else t
        self.nat.check(self.nat.lib().hicu_allreduce(self.h, v.data_ptr(), v.numel(), self.nat.stream_handle()),
                       "allreduce")
        return t

    def exchange(self, ops):
        """ops: [(peer, kind, tensor)], one grouped NCCL round on the current stream."""
        import ctypes

        if not ops:
            return
        arr = (self.nat.HicuP2P * len(ops))()
        for i, (peer, kind, t) in enumerate(ops):
            arr[i].peer, arr[i].kind, arr[i].buf = peer, kind, t.data_ptr()
            arr[i].bytes = t.numel() * t.element_size()
        self.nat.check(self.nat.lib().hicu_halo_exchange(self.h, len(ops), ctypes.cast(arr, ctypes.c_void_p),
                                                         self.nat.stream_handle()), "halo_exchange")

    def close(self):
        if self.h:
            self.nat.lib().hicu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HaloExchange:
    """Exchanges of plane blocks along the sharded axis over
    ``torch.distributed`` (NCCL for CUDA tensors, gloo for CPU tensors).

    Every rank derives the whole exchange pattern from the plans of all ranks:
    each trailing halo run goes to (accumulate) or comes from (refresh) the
    rank owning those planes, which may be several ranks away when shards are
    thinner than the halo, and wraps around on a circular axis.  Received
    partials are added in a fixed (source-rank) order.  With a ``gloo``
    group, device tensors are staged through host memory (gloo moves host
    buffers): the CPU-only multi-rank tests and the single-GPU multi-process
    test of the CUDA backend."""

    def __init__(self, plan: ShardPlan, group=None, native: NativeComm | None = None):
        import torch.distributed as dist

        self.plan = plan
        self.group = group
        self.dist = dist
        self.native = native
        self.host_staged = native is None and dist.get_backend(group) == "gloo"
        self.sends, self.recvs = [], []  # accumulate direction
        for k in range(plan.world):
            for (i0, n, owner, oi0) in plan.for_rank(k).trailing_runs():
                if k == plan.rank:
                    self.sends.append((owner, i0, n, oi0))
                if owner == plan.rank:
                    self.recvs.append((k, oi0, n, i0))
        self.recvs.sort(key=lambda r: (r[0], r[1]))

    def _peer(self, k):
        return k if self.group is None else self.dist.get_global_rank(self.group, k)

    def _run(self, ops):
        if not ops:
            return
        if self.native is not None:
            self.native.exchange(ops)
            return
        for r in self.dist.batch_isend_irecv(ops):
            r.wait()

    def _op(self, kind, t, peer):
        if self.native is not None:
            from . import _native as nat

            return (peer, nat.P2P_SEND if kind == "send" else nat.P2P_RECV, t)
        d = self.dist
        return d.P2POp(d.isend if kind == "send" else d.irecv, t, self._peer(peer), group=self.group)

    def _out(self, t):
        t = t.contiguous()
        return t.cpu() if self.host_staged and t.is_cuda else t

    def _buf(self, like, shape):
        import torch

        dev = "cpu" if self.host_staged else like.device
        return torch.empty(shape, dtype=like.dtype, device=dev)

    def accumulate(self, g_local):
        """Send my trailing halo partials to their owners; add the partials
        other ranks hold of my owned planes into them."""
        import torch

        dist, ax, me = self.dist, self.plan.axis, self.plan.rank
        ops, bufs = [], []
        for (dst, i0, n, oi0) in self.sends:
            if dst == me:
                continue
            ops.append(self._op("send", self._out(g_local.narrow(ax, i0, n)), dst))
        for (src, oi0, n, i0) in self.recvs:
            if src == me:
                bufs.append((oi0, g_local.narrow(ax, i0, n).clone()))
                continue
            shape = list(g_local.shape)
            shape[ax] = n
            buf = self._buf(g_local, shape)
            ops.append(self._op("recv", buf, src))
            bufs.append((oi0, buf))
        self._run(ops)
        for oi0, buf in bufs:
            g_local.narrow(ax, oi0, buf.shape[ax]).add_(buf.to(g_local.device))

    def refresh(self, g_local):
        """Owners send the final values of my trailing halo planes to me."""
        import torch

        dist, ax, me = self.dist, self.plan.axis, self.plan.rank
        ops, fills = [], []
        for (src, oi0, n, i0) in self.recvs:
            if src == me:
                continue
            ops.append(self._op("send", self._out(g_local.narrow(ax, oi0, n)), src))
        for (dst, i0, n, oi0) in self.sends:
            if dst == me:
                fills.append((i0, g_local.narrow(ax, oi0, n).clone()))
                continue
            shape = list(g_local.shape)
            shape[ax] = n
            buf = self._buf(g_local, shape)
            ops.append(self._op("recv", buf, dst))
            fills.append((i0, buf))
        self._run(ops)
        for i0, buf in fills:
            g_local.narrow(ax, i0, buf.shape[ax]).copy_(buf)

    def allreduce_(self, t):
        if self.native is not None:
            return self.native.allreduce_(t)
        if self.host_staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return t
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


def plan_for(dims, kernel, schedule, world: int, rank: int, axis: int = 0) -> ShardPlan:
    """Shard plan along ``axis`` (a spatial axis); every stage must have the
    same region on that axis (C5: readout, axis 0; C4: time, axis 2, whose
    center-out stage windows only x and y)."""
    from .solver import stage_region

    nd = len(dims)
    if not (0 <= axis < nd - 1):
        raise ConfigError(f"cannot shard along axis {axis} (the last axis is the coil axis)")
    regs = [stage_region(dims, kernel, st.region, schedule.circular_axes) for st in schedule.stages]
    ra = {(r.offsets[axis], r.extents[axis]) for r in regs}
    if len(ra) != 1:
        raise ConfigError(f"sharded mode needs the same axis-{axis} region in every stage")
    roff, rext = ra.pop()
    circ = axis in {int(a) % nd for a in schedule.circular_axes}
    return ShardPlan(tuple(dims), kernel.extents[axis], roff, rext, world, rank, axis, circ)


class CudaShardBackend:
    """Local compute of one shard on the current CUDA device through the C ABI."""

    def __init__(self, x0, mask, kernel, schedule, plan: ShardPlan, coil_compress: int | None = None,
                 cov_reduce=None):
        from . import _native as nat
        from .hankel import Region, device_geometry, to_dev
        from .solver import ReconEngine, draw_stage, stage_region

        self.nat = nat
        self.torch = nat.require_cuda()
        torch = self.torch
        self.schedule = schedule
        self.plan = plan
        self.kernel = kernel
        ax = plan.axis
        x0 = np.asarray(x0)
        mask = np.asarray(mask)
        observed = mask == 1
        planes = plan.planes
        xm = np.take(np.where(observed, x0, 0).astype(np.complex64), planes, axis=ax)
        self.mask_np = np.take(observed.astype(np.uint8), planes, axis=ax)
        ldims = plan.local_dims
        self.basis = None
        if coil_compress is not None:
            # distributed SVD coil compression: covariance of the owned planes,
            # summed over ranks, one basis everywhere, applied to the local slab
            from .coil import coil_compress_device

            nc, nv = x0.shape[-1], int(coil_compress)
            xd = to_dev(xm).reshape(-1)
            md = to_dev(self.mask_np, np.uint8).reshape(-1)
            own = [slice(None)] * xm.ndim
            own[ax] = slice(0, plan.owned)
            xo = to_dev(np.ascontiguousarray(xm[tuple(own)])).reshape(-1)
            mo = to_dev(np.ascontiguousarray(self.mask_np[tuple(own)]), np.uint8).reshape(-1)
            y, _, self.basis, _ = coil_compress_device(xd, md, nc, nv, cov_from=(xo, mo), cov_reduce=cov_reduce)
            ldims = ldims[:-1] + (nv,)
            xm = y.reshape(ldims).cpu().numpy()
            self.mask_np = np.ascontiguousarray(self.mask_np[..., :nv])
        circ_local = tuple(a for a in schedule.circular_axes if int(a) % x0.ndim != ax)
        self.regions = []
        for st in schedule.stages:
            rg = stage_region(x0.shape[:-1] + (ldims[-1],), kernel, st.region, schedule.circular_axes)
            offs, exts = list(rg.offsets), list(rg.extents)
            offs[ax], exts[ax] = plan.local_roff0, plan.r1 - plan.r0
            self.regions.append(Region(tuple(offs), tuple(exts), frozenset(int(a) % x0.ndim for a in circ_local)))
        local_sched = schedule
        if len(circ_local) != len(schedule.circular_axes):
            import copy

            local_sched = copy.copy(schedule)
            local_sched.circular_axes = circ_local
        self.eng = ReconEngine(xm, self.mask_np, ldims, kernel, local_sched, self.regions)
        for si, st in enumerate(schedule.stages):
            om, pb = draw_stage(schedule, si, st, kernel.n)
            self.eng.set_host_draws(si, om, pb)
        self.geoms = [device_geometry(kernel, rg, ldims) for rg in self.regions]
        self.sums = torch.zeros(8, dtype=torch.float64, device="cuda")
        # data-consistency mask: bit 1 marks the halo planes (left out of the step sums)
        dcm = self.mask_np.copy()
        sl = [slice(None)] * len(ldims)
        sl[ax] = slice(plan.owned, None)
        dcm[tuple(sl)] |= 2
        self.dc_mask = to_dev(dcm, np.uint8).reshape(-1)
        self.N = int(np.prod(ldims))
        self.dc_parts = torch.zeros(4 * nat.lib().hicu_dc_nparts(self.N), dtype=torch.float64, device="cuda")
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
        """Nystrom on the all-reduced Gram, then the stage driver's closed-form
        complement (hicu_complement_jl): bit-identical on every rank."""
        e, L, nat = self.eng, self.nat.lib(), self.nat
        n, r, ell = e.n, e.r, e.ell
        st = self.schedule.stages[si]
        om, pb = e.stage_data[si]
        nat.check(L.hicu_nystrom(n, ell, r, G.data_ptr(), om[it].data_ptr(), e.V.data_ptr(), e.nys_ws.data_ptr(),
                                 e.nys_bytes, e.status.data_ptr(), self._st()), "nystrom")
        nat.check(L.hicu_complement_jl(n, r, st.gradient_steps * st.p, st.p, e.V.data_ptr(), pb[it].data_ptr(),
                                       e.B.data_ptr(), e.qt32.data_ptr(), e.refl.data_ptr(), e.tau.data_ptr(),
                                       e.flags.data_ptr(), 1e-12, e.status.data_ptr(), self._st()), "complement_jl")

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
        return e.g.view(self.ldims)

    def dc_apply(self, owned_planes):
        """DC on every local sample; the step sums count the owned planes only
        (halo planes carry bit 1 of the DC mask; refresh overwrites them)."""
        e, L = self.eng, self.nat.lib()
        soft = self.schedule.dc_mode == "soft"
        self.nat.check(L.hicu_dc_apply(self.N, e.g.data_ptr(), self.dc_mask.data_ptr(), e.y.data_ptr(),
                                       e.x0.data_ptr() if soft else None, 1 if soft else 0,
                                       float(self.schedule.dc_lambda) if soft else 0.0, self.dc_parts.data_ptr(),
                                       self._st()), "dc_apply")
        self._ndc = self.nat.lib().hicu_dc_nparts(self.N)

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
        y = self.eng.y.view(self.ldims).narrow(pl.axis, 0, pl.owned).cpu().numpy().astype(np.complex128)
        recs = [r.cpu().numpy().reshape(-1, self.nat.REC_SLOTS) for r in self.eng.recs]
        return y, recs


def gather_planes(local_owned, plan: ShardPlan, group=None):
    """All-gather the owned planes of every rank along the sharded axis into
    the full volume (rank order = plane order).  CPU (gloo) or CUDA (NCCL)."""
    import torch
    import torch.distributed as dist

    ax = plan.axis
    t = torch.as_tensor(local_owned)
    maxp = max(plan.P[k + 1] - plan.P[k] for k in range(plan.world))
    shape = list(t.shape)
    shape[ax] = maxp
    pad = torch.zeros(shape, dtype=t.dtype, device=t.device)
    pad.narrow(ax, 0, t.shape[ax]).copy_(t)
    pad_r = torch.view_as_real(pad).contiguous() if pad.is_complex() else pad
    outs = [torch.empty_like(pad_r) for _ in range(plan.world)]
    dist.all_gather(outs, pad_r, group=group)
    blocks = []
    for k in range(plan.world):
        o = torch.view_as_complex(outs[k]) if pad.is_complex() else outs[k]
        blocks.append(o.narrow(ax, 0, plan.P[k + 1] - plan.P[k]))
    return torch.cat(blocks, dim=ax)


def sharded_reconstruct(x0, mask, kernel, schedule, group=None, axis: int = 0, coil_compress: int | None = None,
                        native_comm: bool | None = None):
    """Reconstruct one volume sharded along ``axis`` (C5: readout, 0; C4:
    time, 2) over the ranks of ``group`` (one GPU per rank).  Returns (xhat
    complex128 full volume, records of this rank's run: list per stage of
    [iters*G, 8] arrays).  ``coil_compress=Nv``: distributed SVD coil
    compression first (covariance all-reduced, one basis on every rank);
    ``xhat`` is then in the compressed domain, as hicu_reconstruct's.
    ``native_comm`` (default: with an NCCL group): the library's own NCCL
    communicator carries the halos and all-reduces on the compute stream."""
    import torch.distributed as dist

    from . import _native as nat

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    x0 = np.asarray(x0)
    mask = np.asarray(mask)
    dims = x0.shape if coil_compress is None else x0.shape[:-1] + (int(coil_compress),)
    plan = plan_for(dims, kernel, schedule, world, rank, axis)
    if native_comm is None:
        native_comm = dist.get_backend(group) == "nccl" and bool(nat.lib().hicu_comm_available())
    native = NativeComm(group) if native_comm else None
    halo = HaloExchange(plan, group, native)
    backend = CudaShardBackend(x0, mask, kernel, schedule, plan, coil_compress=coil_compress,
                               cov_reduce=lambda c: halo.allreduce_(torch_view_real(c)))
    y_owned, recs = ShardedReconstruction(backend, plan, halo).run()
    import torch

    yt = torch.from_numpy(y_owned)
    if dist.get_backend(group) != "gloo":
        yt = yt.cuda()
    full = gather_planes(yt, plan, group).cpu().numpy()
    if native is not None:
        native.close()
    if schedule.dc_mode == "hard" and coil_compress is None:
        obs = mask == 1
        full[obs] = np.asarray(x0, np.complex128)[obs]
    return full, recs


def torch_view_real(t):
    return t.view(t.real.dtype) if t.is_complex() else t
