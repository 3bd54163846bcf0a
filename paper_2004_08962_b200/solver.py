"""Staged HICU reconstruction on the B200 — drop-in for ``hicu.hicu_reconstruct``.

Mirrors the reference module ``hicu.solver`` (solver.py): ``StageSpec``,
``SolverSchedule``, ``stage_region``, the record types and
``hicu_reconstruct`` keep their names, arguments, validation and error
classes.  The algorithm is the reference's Algorithm 1 (solver.py:258-398):
per outer iteration a nullspace estimate of the stage region's lifted matrix,
its Householder complement, then ``gradient_steps`` steps each with a fresh
JL compression, a gradient, an exact line search and an update.

B200 execution: all random draws are made on the host up front with the
reference's streams (``RngStream(seed).child(1, stage, it)`` for the sketch,
``child(2, stage, it, step)`` for JL), uploaded once, and each stage runs as
ONE call into the native driver ``hicu_run_stage`` (engine.cu), which
launches Gram -> Nystrom -> Householder -> Q~ and the fused gradient-step
kernels on one CUDA stream with no host synchronisation.  Per-step scalars
live in a device record array that is read once per stage.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _native as nat
from .errors import ConfigError, DegenerateInputError
from .hankel import Counters, KernelMask, MemoryMeter, Region, device_geometry, full_region, to_dev
from .subspace import RngStream, complex_normal

__all__ = [
    "StageSpec",
    "SolverSchedule",
    "stage_region",
    "StepRecord",
    "IterationRecord",
    "ReconReport",
    "hicu_reconstruct",
    "hicu_reconstruct_batch",
    "ReconEngine",
]

_RSVD_STREAM = 1
_JL_STREAM = 2


@dataclass
class StageSpec:
    """One stage (solver.py:51-72): region, compression p, gradient steps per
    nullspace update, iterations."""

    region: object
    p: int
    gradient_steps: int
    iterations: int

    def validate(self) -> None:
        if self.p < 1:
            raise ConfigError("p must be >= 1")
        if self.gradient_steps < 1:
            raise ConfigError("gradient_steps must be >= 1")
        if self.iterations < 1:
            raise ConfigError("iterations must be >= 1")
        if self.p > 32:
            raise ConfigError("p must be <= 32 on the B200 path")


@dataclass
class SolverSchedule:
    """Rank, stages, wrap axes, data consistency, seed (solver.py:75-101)."""

    rank: int
    stages: list
    circular_axes: tuple = ()
    dc_mode: str = "hard"
    dc_lambda: float = 0.0
    seed: int = 0

    def validate(self, kernel: KernelMask, dims) -> list:
        if self.rank < 1:
            raise ConfigError("rank must be >= 1")
        if self.rank >= kernel.n:
            raise ConfigError(f"rank {self.rank} must be below the kernel support size {kernel.n}")
        if not self.stages:
            raise ConfigError("schedule needs at least one stage")
        if self.dc_mode not in ("hard", "soft"):
            raise ConfigError(f"unknown dc_mode {self.dc_mode!r}")
        if self.dc_mode == "soft" and self.dc_lambda <= 0:
            raise ConfigError("soft data consistency needs dc_lambda > 0")
        regions = []
        for stage in self.stages:
            stage.validate()
            regions.append(stage_region(dims, kernel, stage.region, self.circular_axes))
        return regions


def _window_extent(entry, n_d: int, k_d: int, axis: int) -> int:
    """solver.py:104-124 (fractions use Python's round(): banker's rounding)."""
    if entry == "full":
        return n_d
    if isinstance(entry, bool):
        raise ConfigError(f"invalid region entry {entry!r} on axis {axis}")
    if isinstance(entry, (int, np.integer)):
        w = int(entry)
    elif isinstance(entry, (float, Fraction)):
        f = float(entry)
        if not (0.0 < f <= 1.0):
            raise ConfigError(f"region fraction on axis {axis} must be in (0, 1], got {f}")
        w = int(round(f * n_d))
    else:
        raise ConfigError(f"invalid region entry {entry!r} on axis {axis}")
    if w < k_d:
        raise ConfigError(f"stage window {w} on axis {axis} is smaller than the kernel extent {k_d}")
    if w > n_d:
        raise ConfigError(f"stage window {w} on axis {axis} exceeds the array extent {n_d}")
    return w


def stage_region(dims, kernel: KernelMask, fraction, circular_axes=()) -> Region:
    """Centered convolution-output region for one stage (solver.py:127-158).

    The center-out schedule is a restriction of the same operators (kernel
    parameters roff/rext), not a separate code path."""
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    circ = frozenset(int(a) % nd for a in circular_axes)
    if isinstance(fraction, str) and fraction == "full":
        entries = ["full"] * nd
    else:
        entries = list(fraction)
        if len(entries) > nd:
            raise ConfigError(f"region spec has {len(entries)} entries for {nd} axes")
        entries += ["full"] * (nd - len(entries))
    offsets, extents = [], []
    for d, (n_d, k_d) in enumerate(zip(dims, kernel.extents)):
        if k_d > n_d:
            raise ConfigError(f"kernel extent {k_d} exceeds array extent {n_d} on axis {d}")
        if d in circ:
            offsets.append(0)
            extents.append(n_d)
            continue
        entry = "full" if d == nd - 1 else entries[d]
        w = _window_extent(entry, n_d, k_d, d)
        offsets.append((n_d - w) // 2)
        extents.append(w - k_d + 1)
    region = Region(tuple(offsets), tuple(extents), circ)
    region.validate(kernel, dims)
    return region


@dataclass
class StepRecord:
    stage: int
    iteration: int
    step: int
    eta: float
    objective_before: float
    objective_after: float
    seconds: float
    ser_db: float | None = None


@dataclass
class IterationRecord:
    stage: int
    iteration: int
    objective: float | None
    seconds: float
    ser_db: float | None = None
    tail_energy: float | None = None


@dataclass
class ReconReport:
    """Per-run trace (solver.py:161-231) plus B200 extras (``device``,
    ``coil_basis``)."""

    steps: list = field(default_factory=list)
    iterations: list = field(default_factory=list)
    events: list = field(default_factory=list)
    counters: dict = field(default_factory=dict)
    peak_aux_complex: int = 0
    total_seconds: float = 0.0
    device: dict = field(default_factory=dict)
    coil_basis: np.ndarray | None = None

    def to_dict(self) -> dict:
        def _num(v):
            if v is None:
                return None
            if isinstance(v, float) and not np.isfinite(v):
                return "+inf" if v > 0 else "-inf"
            return v

        return {
            "steps": [
                {"stage": s.stage, "iteration": s.iteration, "step": s.step, "eta": s.eta,
                 "objective_before": s.objective_before, "objective_after": s.objective_after,
                 "seconds": s.seconds, "ser_db": _num(s.ser_db)}
                for s in self.steps
            ],
            "iterations": [
                {"stage": i.stage, "iteration": i.iteration, "objective": i.objective, "seconds": i.seconds,
                 "ser_db": _num(i.ser_db), "tail_energy": i.tail_energy}
                for i in self.iterations
            ],
            "events": list(self.events),
            "counters": dict(self.counters),
            "peak_aux_complex": self.peak_aux_complex,
            "total_seconds": self.total_seconds,
            "device": dict(self.device),
        }


class _Stopwatch:
    """Wall clock paused while instrumentation runs (solver.py:234-248)."""

    def __init__(self):
        self.total = 0.0
        self._t0 = time.perf_counter()

    def pause(self) -> float:
        self.total += time.perf_counter() - self._t0
        self._t0 = None
        return self.total

    def resume(self) -> None:
        self._t0 = time.perf_counter()


def _ser_from_parts(parts: np.ndarray) -> float:
    e = math.fsum(parts[0::2].tolist())
    r = math.fsum(parts[1::2].tolist())
    if e == 0.0:
        return float("inf")
    return 20.0 * math.log10(math.sqrt(r) / math.sqrt(e))


def _fill_draws(schedule: SolverSchedule, si: int, stage: StageSpec, n: int, it: int, omega_out, pbig_out):
    """Host draws of one outer iteration with the reference streams
    (solver.py:325-333, subspace.py:112-116, 228): omega (n, l) and pbig
    (n, G*p) with P_j in rows r.. of column block j (rows < r stay zero)."""
    r = schedule.rank
    ell = math.ceil(1.5 * r)
    root = RngStream(schedule.seed)
    G, p = stage.gradient_steps, stage.p
    omega_out[...] = complex_normal(root.child(_RSVD_STREAM, si, it).generator(), (n, ell), 1.0)
    pbig_out[:r, :] = 0
    for j in range(G):
        pbig_out[r:, j * p:(j + 1) * p] = complex_normal(root.child(_JL_STREAM, si, it, j).generator(),
                                                         (n - r, p), 1.0 / p)


def draw_stage(schedule: SolverSchedule, si: int, stage: StageSpec, n: int):
    """All host draws of one stage: omega (iters, n, l), pbig (iters, n, G*p)."""
    ell = math.ceil(1.5 * schedule.rank)
    omega = np.empty((stage.iterations, n, ell), np.complex128)
    pbig = np.zeros((stage.iterations, n, stage.gradient_steps * stage.p), np.complex128)
    for it in range(stage.iterations):
        _fill_draws(schedule, si, stage, n, it, omega[it], pbig[it])
    return omega, pbig


class ReconEngine:
    """Device-resident state for one reconstruction: the iterate, mask, data
    and every scratch buffer, plus one ``hicu_stage_args`` per stage.

    ``run_stage`` issues one native call per stage (or per chunk of
    iterations).  Host draws are written into pinned staging buffers (by
    worker threads in :func:`hicu_reconstruct`) and copied asynchronously on
    the compute stream, so drawing overlaps device execution.  The same
    engine can be re-run (``reset``) for benchmarking without reallocating."""

    def __init__(self, x_init, mask, dims, kernel: KernelMask, schedule: SolverSchedule, regions, reference=None):
        torch = nat.require_cuda()
        self.torch = torch
        self.kernel = kernel
        self.schedule = schedule
        self.regions = regions
        self.dims = tuple(int(d) for d in dims)
        self.N = int(np.prod(self.dims))
        n, r = kernel.n, schedule.rank
        self.n, self.r = n, r
        self.ell = math.ceil(1.5 * r)
        self.soft = schedule.dc_mode == "soft"
        dev = "cuda"
        self.x_init = to_dev(x_init).reshape(-1)
        self.y = self.x_init.clone()
        self.mask = to_dev(mask, np.uint8).reshape(-1)
        self.x0 = self.x_init.clone() if self.soft else None
        self.ref = to_dev(reference).reshape(-1) if reference is not None else None
        self.geoms = [device_geometry(kernel, reg, self.dims) for reg in regions]
        L = nat.lib()
        pmax = max(st.p for st in schedule.stages)
        gmax = max(st.gradient_steps for st in schedule.stages)
        smax = max(reg.s for reg in regions)
        ncp = max(g.conv_nparts for g in self.geoms)
        nsp = max(g.scatter_nparts for g in self.geoms)
        gram_ws = max(int(L.hicu_gram_workspace(g.ref())) for g in self.geoms)
        self.nys_bytes = int(L.hicu_nystrom_workspace(n, self.ell))
        self.gram_bytes = gram_ws
        c128, c64, f64, i32 = torch.complex128, torch.complex64, torch.float64, torch.int32
        self.G = torch.empty((n, n), dtype=c128, device=dev)
        self.gram_ws = torch.empty(max(gram_ws, 8), dtype=torch.uint8, device=dev)
        self.nys_ws = torch.empty(self.nys_bytes, dtype=torch.uint8, device=dev)
        self.V = torch.empty((n, r), dtype=c128, device=dev)
        self.refl = torch.empty(2 * n * r, dtype=c128, device=dev)
        self.tau = torch.empty(r, dtype=c128, device=dev)
        self.flags = torch.empty(r + 1, dtype=i32, device=dev)  # + nullspace_jl gate
        self.status = torch.zeros(1, dtype=i32, device=dev)
        self.B = torch.empty((n, gmax * pmax), dtype=c128, device=dev)
        self.qt32 = torch.empty(gmax * n * pmax, dtype=c64, device=dev)
        self.u = torch.empty(smax * pmax, dtype=c64, device=dev)
        self.g = torch.empty(self.N, dtype=c64, device=dev)
        self.obj_parts = torch.empty(ncp, dtype=f64, device=dev)
        self.dc_parts = torch.empty(4 * nsp, dtype=f64, device=dev)
        self.els_parts = torch.empty(2 * ncp, dtype=f64, device=dev)
        self.ser_stride = 2 * int(L.hicu_ser_nparts(self.N))
        self.t0 = torch.zeros(1, dtype=f64, device=dev)
        self.aux_complex = (n * n + 2 * n * self.ell + 2 * self.ell * self.ell + 2 * n * r + n * gmax * pmax
                            + smax * pmax + self.N)
        ns = len(schedule.stages)
        self.stage_data = [None] * ns
        self.host_draws = [None] * ns
        self.copy_stream = None
        self.upload_events = {}
        self.recs = [None] * ns
        self.sers = [None] * ns
        self.inject = [None] * ns
        self.prof = None
        self.h2d_bytes = 0
        for si, st in enumerate(schedule.stages):
            it, G = st.iterations, st.gradient_steps
            self.stage_data[si] = (torch.empty((it, n, self.ell), dtype=c128, device=dev),
                                   torch.empty((it, n, G * st.p), dtype=c128, device=dev))
            self.recs[si] = torch.zeros(it * G * nat.REC_SLOTS, dtype=f64, device=dev)
            if self.ref is not None:
                self.sers[si] = torch.zeros(it * G * self.ser_stride, dtype=f64, device=dev)
        # the draw buffers are fresh allocations: uploads need only be ordered
        # after this point of the compute stream, not after the stages issued
        # since (waiting on the stream tail serialised every chunk's upload
        # behind the previous chunk's compute)
        self.alloc_event = torch.cuda.Event()
        self.alloc_event.record()

    # -- inputs --------------------------------------------------------------
    def host_draw_buffers(self, si: int):
        """Pinned host staging buffers for stage ``si`` (allocated once)."""
        if self.host_draws[si] is None:
            om, pb = self.stage_data[si]
            self.host_draws[si] = (self.torch.empty(om.shape, dtype=om.dtype, pin_memory=True),
                                   self.torch.empty(pb.shape, dtype=pb.dtype, pin_memory=True))
        return self.host_draws[si]

    def upload_draws(self, si: int, it0: int = 0, it1: int | None = None):
        """Async H2D of the staged draws for iterations [it0, it1) on a
        dedicated copy stream (the copy engine overlaps the compute stream;
        in-stream copies would also break the programmatic-launch chain).
        :meth:`run_stage` makes the compute stream wait for the chunk's event."""
        torch = self.torch
        om_h, pb_h = self.host_draw_buffers(si)
        om, pb = self.stage_data[si]
        it1 = om.shape[0] if it1 is None else it1
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream()
            # iteration slices are disjoint and each is written once, so the only
            # ordering needed is after the buffers' allocation
            self.copy_stream.wait_event(self.alloc_event)
        with torch.cuda.stream(self.copy_stream):
            om[it0:it1].copy_(om_h[it0:it1], non_blocking=True)
            pb[it0:it1].copy_(pb_h[it0:it1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        for it in range(it0, it1):
            self.upload_events[(si, it)] = ev
        self.h2d_bytes += (om_h[it0:it1].numel() + pb_h[it0:it1].numel()) * 16

    def set_host_draws(self, si: int, omega: np.ndarray, pbig: np.ndarray):
        om_h, pb_h = self.host_draw_buffers(si)
        om_h.numpy()[...] = omega
        pb_h.numpy()[...] = pbig
        self.upload_draws(si)

    def set_injected_v(self, si: int, v_all):
        """Lockstep parity: use the given V (iters, n, r) instead of Gram+Nystrom."""
        self.inject[si] = None if v_all is None else to_dev(v_all, np.complex128)

    def reset(self):
        self.y.copy_(self.x_init)
        self.status.zero_()

    def stamp_start(self):
        nat.check(nat.lib().hicu_timestamp(self.t0.data_ptr(), nat.stream_handle()), "timestamp")

    # -- execution -----------------------------------------------------------
    def stage_args(self, si: int, it0: int = 0, iters: int | None = None):
        st = self.schedule.stages[si]
        gm = self.geoms[si]
        iters = st.iterations - it0 if iters is None else iters
        omega, pbig = self.stage_data[si]
        a = nat.HicuStageArgs()
        a.geom = gm.struct
        a.r, a.ell, a.p, a.gsteps, a.iters = self.r, self.ell, st.p, st.gradient_steps, iters
        a.dc_mode = 1 if self.soft else 0
        a.lam = float(self.schedule.dc_lambda) if self.soft else 0.0
        a.householder_tol = 1e-12
        a.N = self.N
        a.y = self.y.data_ptr()
        a.mask = self.mask.data_ptr()
        a.x0 = self.x0.data_ptr() if self.x0 is not None else None
        a.omega = omega[it0].data_ptr() if iters > 0 else omega.data_ptr()
        a.pbig = pbig[it0].data_ptr() if iters > 0 else pbig.data_ptr()
        inj = self.inject[si]
        a.inject_v = inj[it0].data_ptr() if inj is not None and iters > 0 else None
        a.G, a.gram_ws, a.gram_ws_bytes = self.G.data_ptr(), self.gram_ws.data_ptr(), self.gram_bytes
        a.nys_ws, a.nys_ws_bytes = self.nys_ws.data_ptr(), self.nys_bytes
        a.V, a.refl, a.tau = self.V.data_ptr(), self.refl.data_ptr(), self.tau.data_ptr()
        a.flags, a.status = self.flags.data_ptr(), self.status.data_ptr()
        a.B, a.qt32, a.u, a.g = self.B.data_ptr(), self.qt32.data_ptr(), self.u.data_ptr(), self.g.data_ptr()
        a.obj_parts, a.dc_parts, a.els_parts = (self.obj_parts.data_ptr(), self.dc_parts.data_ptr(),
                                                self.els_parts.data_ptr())
        G = st.gradient_steps
        a.rec = self.recs[si].data_ptr() + it0 * G * nat.REC_SLOTS * 8
        if self.ref is not None:
            a.ref = self.ref.data_ptr()
            a.ser_parts = self.sers[si].data_ptr() + it0 * G * self.ser_stride * 8
            a.ser_stride = self.ser_stride
        else:
            a.ref = None
            a.ser_parts = None
            a.ser_stride = 0
        a.prof = self.prof.h if self.prof is not None else None
        return a

    def run_stage(self, si: int, it0: int = 0, iters: int | None = None, stream=None):
        a = self.stage_args(si, it0, iters)
        n_it = self.schedule.stages[si].iterations if iters is None else iters
        cur = stream if stream is not None else self.torch.cuda.current_stream()
        waited = set()
        for it in range(it0, it0 + n_it):
            ev = self.upload_events.pop((si, it), None)
            if ev is not None and id(ev) not in waited:
                cur.wait_event(ev)
                waited.add(id(ev))
        nat.check(nat.lib().hicu_run_stage(ctypes.byref(a), nat.stream_handle(stream)), f"stage {si}")

    def run_all(self, stream=None):
        for si in range(len(self.schedule.stages)):
            self.run_stage(si, stream=stream)

    def check_status(self):
        v = int(self.status.item())
        if v != 0:
            raise DegenerateInputError(
                f"nullspace step failed on the device ({nat.lib().hicu_status_string(v).decode()})")

    def tail_energy(self, kernel: KernelMask, tail_region: Region, r: int) -> float:
        """sum_{j>r} sigma_j^2 of the full-region lifted matrix from its Gram
        matrix (instrumentation; reference oracle.tail_energy_dense)."""
        from .subspace import gram_matrix

        G = gram_matrix(self.y.reshape(self.dims), kernel, tail_region).cpu().numpy()
        lam = np.linalg.eigvalsh(0.5 * (G + G.conj().T))[::-1]
        lam = np.clip(lam, 0.0, None)
        return float(max(np.sum(lam[r:]), 0.0))

    def download(self) -> np.ndarray:
        """complex128 copy of the iterate (pinned staging, multithreaded widening)."""
        return _PINNED.download(self.torch, self.y).reshape(self.dims)


_DRAW_POOL = None


class _PhaseTrace:
    """HICU_E2E_TRACE=1: wall-clock phase marks of hicu_reconstruct on stderr."""

    def __init__(self):
        import os
        import time

        self.on = bool(os.environ.get("HICU_E2E_TRACE"))
        self.t0 = time.perf_counter()
        self.clock = time.perf_counter

    def __call__(self, name):
        if self.on:
            import sys

            print(f"hicu_reconstruct {name}: {1e3 * (self.clock() - self.t0):.2f} ms", file=sys.stderr)


def _draw_pool():
    global _DRAW_POOL
    if _DRAW_POOL is None:
        import concurrent.futures as cf
        import os

        _DRAW_POOL = cf.ThreadPoolExecutor(max_workers=max(1, min(8, len(os.sched_getaffinity(0)))),
                                           thread_name_prefix="hicu-draws")
    return _DRAW_POOL


def _chunks(schedule: SolverSchedule, per_iter: bool):
    """Stage chunks issued to the device one at a time.  The very first chunk
    is a single iteration so the device starts while the host is still
    drawing the later ones."""
    first = True
    for si, st in enumerate(schedule.stages):
        step = 1 if per_iter else max(1, min(8, (st.iterations + 3) // 4))
        it0 = 0
        while it0 < st.iterations:
            n = 1 if first else step
            first = False
            yield si, it0, min(st.iterations, it0 + n)
            it0 += n


class _PinnedPool:
    """Reused pinned host staging buffers for complex64 uploads (allocating
    pinned memory per call cost ~2 ms).

    A buffer is checked out under the lock: it is taken only if no call holds
    it and the device has finished the copy issued from it last time (its
    event has completed); otherwise a new buffer is allocated.  So concurrent
    reconstructions (``hicu_reconstruct_batch`` threads) never share a buffer
    whose copy is still pending.  Idle buffers beyond ``max_idle_bytes`` are
    released (oldest first)."""

    def __init__(self, max_idle_bytes: int = 1 << 31):
        import threading

        self.lock = threading.Lock()
        self.free = []  # [(nbytes, buf, event)] in release order
        self.max_idle = max_idle_bytes

    def _take(self, torch, n):
        with self.lock:
            for i, (nb, b, ev) in enumerate(self.free):
                if b.numel() == n and (ev is None or ev.query()):
                    del self.free[i]
                    return b
        return torch.empty(n, dtype=torch.complex64).pin_memory()

    def _give(self, torch, buf, ev):
        with self.lock:
            self.free.append((buf.numel() * 8, buf, ev))
            idle = sum(e[0] for e in self.free)
            while idle > self.max_idle and len(self.free) > 1:
                idle -= self.free.pop(0)[0]

    def download(self, torch, t):
        """complex128 numpy copy of a complex64 device tensor through a pinned
        buffer (the widening runs on torch's CPU threads)."""
        n = t.numel()
        buf = self._take(torch, n)
        src = t.reshape(-1)
        if n < (1 << 22):
            buf.copy_(src)  # synchronous device-to-host copy on the current stream
            out = buf.to(torch.complex128).numpy()
            self._give(torch, buf, None)
            return out
        # large volumes: the copy goes out in pieces and each piece is widened while the next is
        # still on the bus (419 MB at C5: 17 ms of copy and 13 ms of widening no longer add up)
        pieces = 8
        step = (n + pieces - 1) // pieces
        out = torch.empty(n, dtype=torch.complex128)
        evs = []
        for a in range(0, n, step):
            buf[a:a + step].copy_(src[a:a + step], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            evs.append((a, ev))
        for a, ev in evs:
            ev.synchronize()
            out[a:a + step].copy_(buf[a:a + step])
        self._give(torch, buf, None)
        return out.numpy()

    def upload(self, torch, a):
        a = np.asarray(a)
        n = a.size
        buf = None
        with self.lock:
            for i, (nb, b, ev) in enumerate(self.free):
                if b.numel() == n and (ev is None or ev.query()):
                    buf = b
                    del self.free[i]
                    break
        if buf is None:
            buf = torch.empty(n, dtype=torch.complex64).pin_memory()
        src = np.ascontiguousarray(a)
        if src.dtype in (np.complex64, np.complex128):
            import warnings

            with warnings.catch_warnings():  # read-only caller arrays: torch only reads them here
                warnings.simplefilter("ignore")
                buf.copy_(torch.from_numpy(src).reshape(-1))  # cast + copy on torch's CPU threads
        else:
            np.copyto(buf.numpy().reshape(a.shape), a, casting="unsafe")
        out = buf.to("cuda", non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        with self.lock:
            self.free.append((buf.numel() * 8, buf, ev))
            idle = sum(e[0] for e in self.free)
            while idle > self.max_idle and len(self.free) > 1:
                idle -= self.free.pop(0)[0]
        return out


_PINNED = _PinnedPool()


def _upload_pinned(torch, a):
    """complex64 copy of ``a`` on the device through a pinned staging buffer
    (asynchronous, ordered on the current stream; see :class:`_PinnedPool`)."""
    return _PINNED.upload(torch, a)


def hicu_reconstruct(x0, mask, kernel: KernelMask, schedule: SolverSchedule, reference=None,
                     tail_energy_threshold: int = 2**24, iterate_callback=None, counters: Counters | None = None,
                     meter: MemoryMeter | None = None, *, coil_compress: int | None = None, lockstep_v=None):
    """Run the staged completion on zero-filled observed k-space
    (solver.py:258-398).  Returns ``(xhat, report)``; ``xhat`` is complex128
    like the reference's.  In hard data-consistency mode the observed
    samples of ``xhat`` equal ``x0`` bit-exactly.

    B200 additions (keyword-only): ``coil_compress=Nv`` compresses the coil
    axis to Nv virtual coils on the device first (SVD coil compression; the
    kernel's last extent must then be Nv; ``xhat`` is in the compressed
    domain and ``report.coil_basis`` holds the basis); ``lockstep_v`` is a
    callable ``(stage, it) -> V`` that replaces the nullspace estimate
    (trajectory-parity tests).
    """
    watch = _Stopwatch()
    _tr = _PhaseTrace()
    x0 = np.asarray(x0)
    mask = np.asarray(mask)
    if x0.shape != mask.shape:
        raise ConfigError(f"mask shape {mask.shape} does not match k-space shape {x0.shape}")
    dims = x0.shape if coil_compress is None else x0.shape[:-1] + (int(coil_compress),)
    regions = schedule.validate(kernel, dims)
    for region in regions:
        ell = int(np.ceil(1.5 * schedule.rank))
        if ell > region.s:
            raise ConfigError(f"sketch width {ell} exceeds region size {region.s}; enlarge the stage region")
    if int(np.ceil(1.5 * schedule.rank)) > 256:
        raise ConfigError("rank above 170 is not supported by the device nullspace kernels")
    torch = nat.require_cuda()
    _obs = []

    def observed_host():
        """mask == 1 on the host (a pass over the whole mask): formed only where the host needs it."""
        if not _obs:
            _obs.append(mask == 1)
        return _obs[0]

    basis = None
    h2d = 0
    if coil_compress is not None:
        from .coil import coil_compress_device

        nc, nv = x0.shape[-1], int(coil_compress)
        if not (1 <= nv <= nc) or nc > 32:
            raise ConfigError(f"coil_compress must be in [1, {min(nc, 32)}], got {coil_compress}")
        # virtual coils mix every physical coil, so the sampling pattern must
        # be the same on every coil (the compressed mask is that pattern)
        observed_in = observed_host()
        if not np.array_equal(observed_in, np.broadcast_to(observed_in[..., :1], observed_in.shape)):
            raise ConfigError("coil_compress needs the same sampling mask on every coil")
        # raw k-space through a reused pinned staging buffer; mask_apply
        # (arrays.py:54-67) is fused into the device coil covariance / apply
        xd = _upload_pinned(torch, x0)
        md = to_dev(observed_in.view(np.uint8), np.uint8)
        h2d += xd.numel() * 8 + md.numel()
        _tr("upload issued")
        ydev, mdev, bdev, _ = coil_compress_device(xd.reshape(-1), md.reshape(-1), nc, nv)
        _tr("coil compression issued")
        dims = x0.shape[:-1] + (nv,)
        x_init, mask_dev = ydev, mdev
        ref_dev = None
        if reference is not None:
            rd = to_dev(np.asarray(reference).astype(np.complex64))
            h2d += rd.numel() * 8
            ref_dev = torch.empty(int(np.prod(dims)), dtype=torch.complex64, device="cuda")
            nat.check(nat.lib().hicu_coil_apply(rd.numel() // nc, nc, nv, rd.data_ptr(), None, bdev.data_ptr(),
                                                ref_dev.data_ptr(), None, nat.stream_handle()), "coil_apply")
        basis = bdev  # downloaded after the solve (no synchronisation here)
        x0_exact = None  # observed samples live (in c64) on the device
        exact_on_device = False
    else:
        dims = x0.shape
        # raw k-space (complex64 on the device) and the observed mask through
        # pinned staging; mask_apply (arrays.py:54-67) runs on the device.  The
        # caller's x0 itself (no copy) re-imposes the observed samples
        # bit-exactly on return.
        x0_exact = x0
        _tr("validated")
        xd = _upload_pinned(torch, x0)
        _tr("k-space upload issued")
        if mask.dtype in (np.uint8, np.bool_):
            # the raw mask bytes go up as they are; mask == 1 (arrays.py:54-67) is taken on the device
            md = (to_dev(mask.view(np.uint8), np.uint8).reshape(-1) == 1).to(torch.uint8)
        else:
            md = to_dev(observed_host().view(np.uint8), np.uint8).reshape(-1)
        _tr("mask uploaded")
        x_init = torch.where(md.bool(), xd, torch.zeros((), dtype=xd.dtype, device=xd.device))
        mask_dev = md
        # complex64 input: its observed samples are exact on the device, so the
        # result is assembled there (no host pass over the volume)
        exact_on_device = x0.dtype == np.complex64
        ref_dev = None if reference is None else np.asarray(reference).astype(np.complex64)
        h2d += xd.numel() * 8 + md.numel() + (0 if ref_dev is None else ref_dev.nbytes)
    counters = counters if counters is not None else Counters()
    meter = meter if meter is not None else MemoryMeter()
    report = ReconReport()
    eng = ReconEngine(x_init, mask_dev, dims, kernel, schedule, regions, ref_dev)
    _tr("engine")
    meter.alloc(eng.aux_complex)
    tail_region = full_region(dims, kernel, schedule.circular_axes)
    log_tail = 0 < tail_energy_threshold and tail_region.s * kernel.n <= tail_energy_threshold
    per_iter = log_tail or iterate_callback is not None
    if lockstep_v is not None:
        for si, stage in enumerate(schedule.stages):
            eng.set_injected_v(si, np.stack([np.asarray(lockstep_v(si, it), np.complex128)
                                             for it in range(stage.iterations)]))
    # host draws (reference streams) on worker threads, overlapped with the device
    pool = _draw_pool()
    futures = []
    for si, it0, it1 in _chunks(schedule, per_iter):
        om_h, pb_h = eng.host_draw_buffers(si)
        om_np, pb_np = om_h.numpy(), pb_h.numpy()
        st = schedule.stages[si]
        futs = [pool.submit(_fill_draws, schedule, si, st, kernel.n, it, om_np[it], pb_np[it])
                for it in range(it0, it1)]
        futures.append((si, it0, it1, futs))
    _tr("setup")
    eng.stamp_start()
    tails = {}
    for si, it0, it1, futs in futures:
        for f in futs:
            f.result()
        eng.upload_draws(si, it0, it1)
        eng.run_stage(si, it0, it1 - it0)
        if not per_iter:
            continue
        torch.cuda.current_stream().synchronize()
        watch.pause()
        eng.check_status()
        if log_tail:
            tails[(si, it0)] = eng.tail_energy(kernel, tail_region, schedule.rank)
        if iterate_callback is not None:
            xi = eng.download()
            if schedule.dc_mode == "hard" and x0_exact is not None:
                np.copyto(xi, x0_exact, where=observed_host())
            iterate_callback(si, it0, xi)
        watch.resume()
    _tr("issued")
    if schedule.dc_mode == "hard" and exact_on_device:
        eng.y.copy_(torch.where(md.bool(), xd, eng.y))  # observed samples: the caller's, exactly
    torch.cuda.current_stream().synchronize()
    _tr("device done")
    xhat = eng.download()
    _tr("download")
    total = watch.pause()
    eng.check_status()
    # ---- records (one device->host read per stage) ----
    t0 = float(eng.t0.item())
    d2h = xhat.size * 8
    for si, stage in enumerate(schedule.stages):
        rec = eng.recs[si].cpu().numpy().reshape(stage.iterations, stage.gradient_steps, nat.REC_SLOTS)
        d2h += rec.nbytes
        sers = None
        if eng.ref is not None:
            sers = eng.sers[si].cpu().numpy().reshape(stage.iterations, stage.gradient_steps, eng.ser_stride)
        p = stage.p
        for it in range(stage.iterations):
            last_obj = None
            last_sec = 0.0
            last_ser = None
            for j in range(stage.gradient_steps):
                rj = rec[it, j]
                sec = max((rj[nat.REC_TIME] - t0) * 1e-9, 0.0)
                ser = _ser_from_parts(sers[it, j]) if sers is not None else None
                counters.forward += p
                counters.kspace_scatter += p
                if rj[nat.REC_GNORM2] > 0.0:
                    counters.forward += p
                if rj[nat.REC_DEGENERATE] != 0.0:
                    report.events.append({"stage": si, "iteration": it, "step": j, "reason": "degenerate-direction"})
                    report.steps.append(StepRecord(si, it, j, 0.0, float(rj[nat.REC_OBJ]), float(rj[nat.REC_OBJ]),
                                                   sec, ser))
                else:
                    report.steps.append(StepRecord(si, it, j, float(rj[nat.REC_ETA]), float(rj[nat.REC_OBJ]),
                                                   float(rj[nat.REC_OBJ_AFTER]), sec, ser))
                last_obj = float(rj[nat.REC_OBJ_AFTER])
                last_sec, last_ser = sec, ser
            if lockstep_v is None:
                counters.gram += 1
            report.iterations.append(IterationRecord(si, it, last_obj, last_sec, last_ser, tails.get((si, it))))
    if schedule.dc_mode == "hard" and x0_exact is not None and not exact_on_device:
        np.copyto(xhat, x0_exact, where=observed_host())
    report.total_seconds = total
    report.counters = counters.snapshot()
    report.peak_aux_complex = meter.peak
    meter.free(eng.aux_complex)
    report.device = {"name": torch.cuda.get_device_name(),
                     "nullspace": "gram+nystrom (canonical phases)" if lockstep_v is None else "injected",
                     "precision": "c64 data, fp32 FMA, fp64 reductions and nullspace",
                     "h2d_bytes": int(h2d + eng.h2d_bytes), "d2h_bytes": int(d2h)}
    report.coil_basis = None if basis is None else basis.cpu().numpy()
    _tr("end")
    return xhat, report


def hicu_reconstruct_batch(x0s, masks, kernel: KernelMask, schedule: SolverSchedule, *, concurrency: int = 8,
                           **kw):
    """Independent reconstructions (the slices of a multi-slice exam, C3)
    run concurrently on ``concurrency`` CUDA streams of the current device;
    returns ``[(xhat, report), ...]`` in input order.

    Each reconstruction is exactly :func:`hicu_reconstruct` (results are
    bit-identical to running them one after another: every kernel is
    deterministic and nothing is shared between streams).  Concurrency lets one
    slice's nullspace step — a chain of single-CTA fp64 kernels — run on a few
    SMs while other slices' convolutions fill the rest of the GPU (SURVEY §8e:
    "batch K1/K2 across the slices on each GPU")."""
    import concurrent.futures as cf

    torch = nat.require_cuda()
    n = len(x0s)
    if len(masks) != n:
        raise ConfigError("need one mask per slice")
    if n == 0:
        return []
    lanes = max(1, min(int(concurrency), n))
    dev = torch.cuda.current_device()
    streams = [torch.cuda.Stream(device=dev) for _ in range(lanes)]
    out = [None] * n

    def lane(k):
        with torch.cuda.device(dev), torch.cuda.stream(streams[k]):
            for i in range(k, n, lanes):
                out[i] = hicu_reconstruct(x0s[i], masks[i], kernel, schedule, **kw)

    with cf.ThreadPoolExecutor(max_workers=lanes, thread_name_prefix="hicu-batch") as ex:
        for f in [ex.submit(lane, k) for k in range(lanes)]:
            f.result()
    return out
