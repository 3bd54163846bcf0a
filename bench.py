"""HICU B200 benchmark (driver contract: one JSON line on rank 0).

``--config`` picks the BASELINE.json configuration; the default is C5
(configs[4]), the largest configuration that fits one B200: one 256x160x160
volume, 8 coils, 2D Poisson-disc R=5, SNR 30 dB, 5x5x5x8 kernel (n = 1000),
rank 120 (l = 180), p = 8, G = 5, 40 outer iterations.  metric = HICU outer
iterations per second (BASELINE.json "HICU iters/s").

A *step* is one pass of the hot path over the input:
* C5: one outer iteration over the whole volume (Gram + nullspace + G
  gradient steps), the steps walking through the 40-iteration schedule;
* C1 / C2 / C4: one full reconstruction (all stages and iterations);
* C3: one full reconstruction of this rank's share of the 64 slices
  (independent slices on 4 concurrent CUDA streams).

* ``value``: device-resident inputs (k-space, mask and all host-seeded
  sketch / JL draws already in HBM); CUDA events on the compute stream,
  barrier + synchronize around each step, max over ranks.  L2: the C5 inputs
  (419 MB k-space) exceed the 126 MB L2; for the smaller configs a 256 MiB
  buffer is written between steps (untimed).
* ``e2e``: the public API ``hicu_reconstruct`` (C3: ``reconstruct_slices``;
  C5 at N > 1: ``sharded_reconstruct``) from host numpy arrays, every
  host->device and device->host copy inside the timed region; the full
  schedule (C5: all 40 iterations).
* ``roofline``: the dominant tensor-core kernel class from the native
  CUDA-event profiler over one extra step, against the measured TF32 peak
  / 3 (3xTF32); ``roofline_all`` lists every class.
* ``cpu_baseline`` (rank 0, N = 1): the reference package itself
  (``baseline/_ref/hicu``, its ``hicu_reconstruct``; the numpy oracle port
  when the install is absent) on a bounded sample: one outer iteration per
  stage on an axis-0 slab of the input, extrapolated linearly in the region
  rows to the full config (the s-independent Householder + JL time measured
  separately and not scaled); 1 thread and all host threads.
* ``--impl reference``: the same reference sampler as the timed arm.

N > 1 (torchrun, NCCL): C5 one volume sharded along the readout axis with
(K0-1)-plane halos, the Gram and the line-search scalars all-reduced (strong
scaling); C4 the series sharded along time with multi-neighbour halos and a
distributed coil compression (strong scaling); C3 the 64 slices partitioned
over ranks (strong scaling); C1 / C2 replicas (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")

DEFAULT_CONFIG = "C5"


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _spec(name):
    from paper_2004_08962_b200.synthetic import CONFIGS

    return CONFIGS[name]


WORKLOAD_TEXT = {
    "C1": "C1 (BASELINE.json configs[0]): 128x128, 8 coils, 2D VD random mask R=3, SNR 30 dB, kernel 5x5x8 (n=200), "
          "rank 40, 50 iterations, p=8, G=5",
    "C2": "C2 (BASELINE.json configs[1]): 256x256, 16->8 coils (device SVD coil compression), 1D VD phase-encode "
          "mask R=4, SNR 30 dB, kernel 5x5x8 (n=200), rank 60, stages 64^2/128^2/full x 25/25/50, p=8, G=5",
    "C3": "C3 (BASELINE.json configs[2]): 64 slices of 320x320, 16->10 coils (device SVD coil compression), "
          "per-slice 1D random mask R=4, kernel 7x7x10 (n=490), rank 100, 20 iterations, p=10, G=5",
    "C4": "C4 (BASELINE.json configs[3]): 192x144x25 cine, 12->8 coils (device SVD coil compression), per-frame "
          "VD phase-encode mask R=6, kernel 5x5x5x8 (n=1000), rank 150, stages [48,36,full]/full x 50/10, p=8, G=5",
    "C5": "C5 (BASELINE.json configs[4]): 256x160x160 volume, 8 coils, 2D Poisson-disc R=5 on the phase/partition "
          "plane, SNR 30 dB, kernel 5x5x5x8 (n=1000), rank 120, 40 iterations, p=8, G=5",
}


def workload_config(name, world):
    spec = _spec(name)
    par = {"C5": f"readout-sharded volume over {world} GPU(s) (halo + NCCL all-reduce)" if world > 1 else "1 GPU",
           "C4": f"time-sharded series over {world} GPU(s) (multi-neighbour halos + NCCL all-reduce)"
           if world > 1 else "1 GPU",
           "C3": f"64 slices partitioned over {world} GPU(s), no collective"}.get(
        name, "replicas (one instance per GPU, no collective)" if world > 1 else "1 GPU")
    return {
        "workload": WORKLOAD_TEXT[name],
        "step": "one outer iteration of the whole volume" if name == "C5" else (
            "one full reconstruction of this rank's slices" if name == "C3" else "one full reconstruction"),
        "iterations_per_reconstruction": spec.iterations,
        "kernel": list(spec.kernel), "rank": spec.rank,
        "stages": [[s[0], s[1], s[2], s[3]] for s in spec.stages],
        "l2": "inputs larger than L2 (419 MB k-space)" if name == "C5" else
              "flushed between steps (256 MiB device write, untimed)",
        "parallelism": par,
    }


# ---------------------------------------------------------------------------
# CPU legs: the reference package (baseline/_ref) or the oracle port
# ---------------------------------------------------------------------------


def _reference_module():
    """(module, kind): the installed reference package, else the oracle port."""
    if os.path.isdir(os.path.join(REF_INSTALL, "hicu")):
        if REF_INSTALL not in sys.path:
            sys.path.insert(0, REF_INSTALL)
        import hicu

        return hicu, "reference"
    from oracle import hicu_oracle

    return hicu_oracle, "port"


_HOST_CACHE = {}


def _compressed_host_input(name, scale=1.0):
    """(x0, mask, coil-compression seconds) as the CPU path receives it: coil
    compression is not part of the reference, so the oracle's
    restatement runs first and is timed separately.  The synthetic k-space is
    generated once per process (C5 takes ~16 s)."""
    from oracle import hicu_oracle as O
    from paper_2004_08962_b200.synthetic import make_config

    spec = _spec(name)
    key = (name, scale)
    if key not in _HOST_CACHE:
        _HOST_CACHE[key] = make_config(name, scale=scale)
    ksp, mask, x0 = _HOST_CACHE[key]
    t = 0.0
    if spec.coils_out != spec.coils_in:
        t0 = time.perf_counter()
        xc, mc, _ = O.coil_compress(x0, mask, spec.coils_out)
        t = time.perf_counter() - t0
        x0, mask = xc.astype(np.complex64), mc
    return x0, mask, t


def _run_cpu_iteration(mod, kind, x0, mask, kext, region, p, G, rank, circular):
    """One outer iteration (nullspace + G gradient steps) of the CPU path;
    returns seconds (the reference's own clock, report.total_seconds)."""
    if kind == "reference":
        kern = mod.KernelMask.full(tuple(kext))
        sched = mod.SolverSchedule(rank=rank, stages=[mod.StageSpec(region, p, G, 1)], circular_axes=tuple(circular),
                                   seed=0)
        _, rep = mod.hicu_reconstruct(x0, mask, kern, sched, tail_energy_threshold=0)
        return rep.total_seconds
    t = time.perf_counter()
    mod.hicu_reconstruct(x0, mask, tuple(kext), [(region, p, G, 1)], rank, circular=tuple(circular), seed=0)
    return time.perf_counter() - t


def _const_seconds(mod, kind, n, r, p, G):
    """s-independent part of an iteration: Householder completion + G JL draws."""
    rng = np.random.default_rng(0)
    v, _ = np.linalg.qr(rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r)))
    t = time.perf_counter()
    if kind == "reference":
        from hicu.subspace import RngStream, householder_nullspace, jl_compress

        q = householder_nullspace(v).q
        for j in range(G):
            jl_compress(q, p, RngStream(0, (2, 0, 0, j)))
    else:
        q = mod.householder_nullspace(v)
        for j in range(G):
            mod.jl_compress(q, p, 0, (2, 0, 0, j))
    return time.perf_counter() - t


def reference_sample(name, threads, budget=1.2e7):
    """Bounded CPU sample of one config: per stage one outer iteration on an
    axis-0 slab holding about budget/n region rows (the whole input when it
    is smaller), extrapolated linearly in region rows to the stage's full
    region; returns (estimated seconds per step, details)."""
    from threadpoolctl import threadpool_limits

    from paper_2004_08962_b200.hankel import KernelMask
    from paper_2004_08962_b200.solver import stage_region

    mod, kind = _reference_module()
    spec = _spec(name)
    x0, mask, t_cc = _compressed_host_input(name)
    kern = KernelMask.full(spec.kernel)
    n, k0 = kern.n, spec.kernel[0]
    ell = math.ceil(1.5 * spec.rank)
    per_stage = []
    with threadpool_limits(threads):
        t_const = None
        for si, (region, p, G, iters) in enumerate(spec.stages):
            reg = stage_region(x0.shape, kern, region, spec.circular_axes)
            s_full = reg.s
            rows_per_plane = s_full // reg.extents[0]
            want = max(ell, int(budget / n))
            planes = min(reg.extents[0], max(1, -(-want // rows_per_plane)))
            if planes < reg.extents[0]:
                # slab of `planes` output planes (+ K0-1 halo) centred in the stage window
                lo = reg.offsets[0] + (reg.extents[0] - planes) // 2
                xs = np.ascontiguousarray(x0[lo:lo + planes + k0 - 1])
                ms = np.ascontiguousarray(mask[lo:lo + planes + k0 - 1])
                reg_s = "full" if region == "full" else ["full"] + list(region[1:])
                s_slab = planes * rows_per_plane
            else:
                xs, ms, reg_s, s_slab = x0, mask, region, s_full
            t_it = _run_cpu_iteration(mod, kind, xs, ms, spec.kernel, reg_s, p, G, spec.rank, spec.circular_axes)
            if s_slab < s_full:
                if t_const is None:
                    t_const = _const_seconds(mod, kind, n, spec.rank, p, G)
                t_full = t_const + max(t_it - t_const, 0.0) * s_full / s_slab
            else:
                t_full = t_it
            per_stage.append({"stage": si, "rows_full": s_full, "rows_sample": s_slab, "sample_s": t_it,
                              "iteration_s_est": t_full, "iterations": iters})
    if name == "C5":
        est = per_stage[0]["iteration_s_est"]           # one step = one outer iteration
    else:
        est = t_cc + sum(st["iteration_s_est"] * st["iterations"] for st in per_stage)
        if name == "C3":
            est *= spec.slices
    return est, {"kind": kind, "coil_compression_s": t_cc, "stages": per_stage, "const_s": t_const,
                 "threads": threads}


def _step_iterations(name):
    spec = _spec(name)
    if name == "C5":
        return 1
    if name == "C3":
        return spec.iterations * spec.slices
    return spec.iterations


def _sample_text(name, det):
    st = det["stages"]
    parts = [f"stage {s['stage']}: one outer iteration on {s['rows_sample']} of {s['rows_full']} region rows" for s in st]
    extra = " (C3: one slice, x64 slices)" if name == "C3" else ""
    return ("; ".join(parts) + ", extrapolated linearly in region rows (Householder+JL time unscaled)"
            + (", + oracle coil compression" if det["coil_compression_s"] else "") + extra)


def run_reference(args):
    """Reference arm: the reference package's CPU path, all host threads,
    bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    threads = _host_threads()
    for _ in range(args.warmup):
        reference_sample(name, threads)
    est_total = 0.0
    det = None
    for _ in range(args.steps):
        est, det = reference_sample(name, threads)
        est_total += est
    units = _step_iterations(name) * args.steps
    value = units / est_total
    line = {
        "metric": "HICU iters/s", "value": value, "unit": "iters/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * est_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": workload_config(name, 1), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": det["kind"],
                         "sample": _sample_text(name, det), "cpu": _cpu_model(), "last_sample": det},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = f"/tmp/hicu_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "100"], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        try:
            os.unlink(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


class DeviceWorkload:
    """Device-resident inputs + engines for one config on this rank, and a
    ``step()`` that issues one step on the current stream."""

    def __init__(self, name, world, rank, group=None):
        import torch

        import paper_2004_08962_b200 as H
        from paper_2004_08962_b200.coil import coil_compress_device
        from paper_2004_08962_b200.hankel import to_dev
        from paper_2004_08962_b200.solver import ReconEngine, draw_stage
        from paper_2004_08962_b200.synthetic import make_config

        self.torch, self.H = torch, H
        self.name, self.world, self.rank = name, world, rank
        spec = self.spec = _spec(name)
        self.kernel = H.KernelMask.full(spec.kernel)
        self.sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages],
                                      circular_axes=spec.circular_axes, seed=0)
        self.it = 0
        self.sharded = None
        if name == "C3":
            from paper_2004_08962_b200.parallel import partition_slices

            self.slices = list(partition_slices(spec.slices, world, rank))
        else:
            self.slices = [rank if world > 1 and name not in ("C4", "C5") else 0]
        self.host = {s: make_config(name, slice_index=s) for s in self.slices}
        nc, nv = spec.coils_in, spec.coils_out
        self.engines = []
        self.resets = []
        if name in ("C4", "C5") and world > 1:
            # one volume sharded over the ranks: readout (C5) or time (C4, with the
            # distributed coil compression: covariance all-reduced, one basis)
            from paper_2004_08962_b200.parallel import (CudaShardBackend, HaloExchange, ShardedReconstruction,
                                                        plan_for, torch_view_real)

            ksp, mask, x0 = self.host[0]
            self.axis = 2 if name == "C4" else 0
            cc = None if nv == nc else nv
            dims = x0.shape[:-1] + (nv,)
            plan = plan_for(dims, self.kernel, self.sched, world, rank, self.axis)
            from paper_2004_08962_b200 import _native as nat
            from paper_2004_08962_b200.parallel import NativeComm

            # halos and all-reduces through the library's own NCCL communicator on the compute stream
            native = NativeComm(group) if nat.lib().hicu_comm_available() else None
            halo = HaloExchange(plan, group, native)
            backend = CudaShardBackend(x0, mask, self.kernel, self.sched, plan, coil_compress=cc,
                                       cov_reduce=lambda c: halo.allreduce_(torch_view_real(c)))
            self.sharded = ShardedReconstruction(backend, plan, halo)
            self.engines = [backend.eng]
            self.resets = [(backend.eng.y, backend.eng.y.clone())]
            self.dims = dims
            return
        for s in self.slices:
            ksp, mask, x0 = self.host[s]
            xd = to_dev(x0).reshape(-1)
            md = to_dev(mask, np.uint8).reshape(-1)
            if nv != nc:
                y, m, _, _ = coil_compress_device(xd, md, nc, nv)
            else:
                y, m = xd, md
            dims = x0.shape[:-1] + (nv,)
            regions = self.sched.validate(self.kernel, dims)
            eng = ReconEngine(y, m, dims, self.kernel, self.sched, regions)
            for si, st in enumerate(self.sched.stages):
                om, pb = draw_stage(self.sched, si, st, self.kernel.n)
                eng.set_host_draws(si, om, pb)
            self.engines.append(eng)
            self.resets.append((xd, md))
            self.dims = dims
        self.streams = [torch.cuda.Stream() for _ in range(min(C3_LANES, len(self.engines)))] if name == "C3" else None

    def step(self):
        torch = self.torch
        spec = self.spec
        if self.sharded is not None:
            if self.name == "C5":
                it = self.it % spec.stages[0][3]
                if it == 0:
                    self.resets[0][0].copy_(self.resets[0][1])
                self.sharded.run_iteration(0, it)
                self.it += 1
                return
            self.resets[0][0].copy_(self.resets[0][1])  # C4: one step = the whole schedule
            for si, st in enumerate(spec.stages):
                for it in range(st[3]):
                    self.sharded.run_iteration(si, it)
            return
        if self.name == "C5":
            eng = self.engines[0]
            it = self.it % spec.stages[0][3]
            if it == 0:
                eng.y.copy_(eng.x_init)
                eng.status.zero_()
            eng.run_stage(0, it, 1)
            self.it += 1
            return
        from paper_2004_08962_b200.coil import coil_compress_device

        nc, nv = spec.coils_in, spec.coils_out

        def one(eng, xd, md):
            if nv != nc:
                y, _, _, _ = coil_compress_device(xd, md, nc, nv)
                eng.y.copy_(y)
            else:
                eng.y.copy_(eng.x_init)
            eng.status.zero_()
            eng.run_all()

        if self.streams is None:
            for eng, (xd, md) in zip(self.engines, self.resets):
                one(eng, xd, md)
            return
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        for k, (eng, (xd, md)) in enumerate(zip(self.engines, self.resets)):
            with torch.cuda.stream(self.streams[k % len(self.streams)]):
                one(eng, xd, md)
        for s in self.streams:
            cur.wait_stream(s)

    def check(self):
        for e in self.engines:
            e.check_status()

    def set_prof(self, prof):
        if self.sharded is not None:
            return
        for e in self.engines:
            e.prof = prof

    def e2e(self, group=None):
        """One call of the public API from host arrays; returns (seconds,
        iterations, h2d bytes, d2h bytes)."""
        H = self.H
        spec = self.spec
        cc = None if spec.coils_out == spec.coils_in else spec.coils_out
        t = time.perf_counter()
        if self.sharded is not None:
            from paper_2004_08962_b200.parallel import sharded_reconstruct

            ksp, mask, x0 = self.host[0]
            xhat, _ = sharded_reconstruct(x0, mask, self.kernel, self.sched, group=group, axis=self.axis,
                                          coil_compress=cc)
            dt = time.perf_counter() - t
            return dt, spec.iterations, x0.nbytes // self.world + mask.nbytes // self.world, xhat.nbytes // self.world
        if self.name == "C3":
            from paper_2004_08962_b200.parallel import reconstruct_slices

            n_all = spec.slices  # this rank holds only its block; reconstruct_slices indexes that block
            xl = [self.host[i][2] if i in self.host else None for i in range(n_all)]
            ml = [self.host[i][1] if i in self.host else None for i in range(n_all)]
            out = reconstruct_slices(xl, ml, self.kernel, self.sched, rank=self.rank, world=self.world,
                                     concurrency=C3_LANES, tail_energy_threshold=0, coil_compress=cc)
            dt = time.perf_counter() - t
            h2d = sum(r.device["h2d_bytes"] for _, r in out.values())
            d2h = sum(r.device["d2h_bytes"] for _, r in out.values())
            return dt, spec.iterations * len(out), h2d, d2h
        ksp, mask, x0 = self.host[self.slices[0]]
        _, rep = H.hicu_reconstruct(x0, mask, self.kernel, self.sched, tail_energy_threshold=0, coil_compress=cc)
        dt = time.perf_counter() - t
        return dt, spec.iterations, rep.device["h2d_bytes"], rep.device["d2h_bytes"]


# C3: independent slices in flight on one GPU (CUDA streams); the nullspace
# kernels are single-CTA / 8-CTA-cluster latency chains, so more slices in
# flight fill more SMs
C3_LANES = int(os.environ.get("HICU_C3_LANES", "16"))


def _work_per_step(dw):
    """Algorithmic work of the kernel classes in one step: real
    flops per class, update bytes; ``gram_path`` is the Gram the library ran
    ("lag": fp32 lag correlations, whose executed flops are counted, and the
    dense-equivalent 4 s n (n+1) is reported beside them)."""
    from paper_2004_08962_b200 import _native as nat

    spec = dw.spec
    n = dw.kernel.n
    dims = dw.dims if dw.sharded is None else dw.sharded.b.ldims
    regions = dw.engines[0].regions
    geoms = dw.engines[0].geoms
    N = int(np.prod(dims))
    tot = {"gram": 0.0, "gram_dense_equiv": 0.0, "conv_fwd": 0.0, "scatter": 0.0, "conv_els": 0.0,
           "update_bytes": 0.0}
    paths = set()
    for st, reg, gm in zip(spec.stages, regions, geoms):
        s, p, G = reg.s, st[1], st[2]
        iters = 1 if dw.name == "C5" else st[3]
        path = nat.GRAM_PATHS[int(nat.lib().hicu_gram_path(gm.ref()))]
        if path == "lag" and nat.lib().hicu_gram_lag_uses_tensor_cores(gm.ref()):
            path = "lag-tc"
        paths.add(path)
        tot["gram"] += float(nat.lib().hicu_gram_flops(gm.ref())) * iters
        tot["gram_dense_equiv"] += 4.0 * s * n * (n + 1) * iters
        for k in ("conv_fwd", "scatter", "conv_els"):
            tot[k] += 8.0 * s * n * p * G * iters
        tot["update_bytes"] += 25.0 * N * G * iters
    mult = len(dw.engines)
    out = {k: v * mult for k, v in tot.items()}
    out["gram_path"] = "/".join(sorted(paths))
    return out


def _load_json(path, default=None):
    try:
        return json.load(open(os.path.join(ROOT, path)))
    except (OSError, ValueError):
        return default


def roofline(kinds, work, peaks, sm_mhz=None, profiled=True):
    # The tensor-core classes compute FP32-grade products as three fp16 MMA
    # products (hi*hi + hi*lo + lo*hi, kind::f16, fp32 accumulation), so their
    # peak is the measured dense 16-bit tensor rate / 3 (MEASURED_PEAKS.json:
    # cuBLAS bf16; f16 runs at the same rate).  The round-1 3xTF32 figure
    # (measured TF32 / 3) is kept beside it for comparison.
    tf32 = _load_json("profiles/tf32_peak_r01.json", {"tf32_tflops": 749.4})
    tf32_peak = tf32["tf32_tflops"] / 3.0
    f16_peak = peaks.get("bf16_tflops", 1629.9) / 3.0
    hbm = peaks.get("hbm_gbs", 6548.2)
    # CUDA-core fp32 peak (FFMA2: 148 SMs x 128 lanes x 2 flop at the max SM clock)
    fp32_peak = 148 * 128 * 2 * (peaks.get("sm_max_mhz", 1965.0) * 1e6) / 1e12
    ncu = {rec["kernel"]: rec for rec in _load_json("profiles/r02_ncu_full.json", [])}
    ncu_name = {"gram": "lagtc_core_kernel", "conv_fwd": "conv_tri_kernel<0", "scatter": "conv_tri_kernel<2",
                "conv_els": "conv_tri_kernel<1", "update": "update_kernel"}

    def traffic(kind):
        if not profiled:  # the committed ncu captures are of the C5 workload
            return None
        for k, rec in ncu.items():
            if ncu_name.get(kind, "@") in k and rec.get("dram_read_bytes") is not None:
                return rec["dram_read_bytes"] + (rec.get("dram_write_bytes") or 0.0)
        return None

    ms_by = {k: v["ms"] for k, v in kinds.items()}
    roof_all = {}
    for k in ("gram", "conv_fwd", "scatter", "conv_els"):
        if ms_by.get(k, 0) <= 0:
            continue
        nl = max(1, kinds[k]["launches"])
        ach = work[k] / (ms_by[k] * 1e-3) / 1e12
        if k == "gram" and work.get("gram_path") == "lag-tc":
            roof_all[k] = {"bound": "tensor", "achieved": ach, "peak": f16_peak, "unit": "TFLOP/s",
                           "frac": ach / f16_peak, "frac_vs_3xtf32_peak": ach / tf32_peak, "traffic": traffic(k),
                           "launches": nl, "avg_launch_ms": ms_by[k] / nl, "flops_per_launch_avg": work[k] / nl,
                           "path": "lag Gram, core class on tcgen05 (lagtc_core_kernel, polyphase line pairs): "
                                   "useful flops of the lag correlations over the whole Gram (prep, core, "
                                   "edges, reduce, assemble)",
                           "dense_equivalent_tflops": work["gram_dense_equiv"] / (ms_by[k] * 1e-3) / 1e12}
            continue
        if k == "gram" and work.get("gram_path") == "lag":
            roof_all[k] = {"bound": "fp32 (CUDA-core FFMA2)", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                           "frac": ach / fp32_peak, "traffic": traffic(k), "launches": nl,
                           "avg_launch_ms": ms_by[k] / nl, "flops_per_launch_avg": work[k] / nl,
                           "path": "lag Gram (gram_lag.cu): executed fp32 flops of the lag correlations",
                           "dense_equivalent_tflops": work["gram_dense_equiv"] / (ms_by[k] * 1e-3) / 1e12}
            continue
        roof_all[k] = {"bound": "tensor", "achieved": ach, "peak": f16_peak, "unit": "TFLOP/s",
                       "frac": ach / f16_peak, "frac_vs_3xtf32_peak": ach / tf32_peak, "traffic": traffic(k),
                       "launches": nl,
                       "avg_launch_ms": ms_by[k] / nl, "flops_per_launch_avg": work[k] / nl}
    if ms_by.get("update", 0) > 0:
        ach = work["update_bytes"] / (ms_by["update"] * 1e-3) / 1e9
        roof_all["update"] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                              "traffic": traffic("update"), "launches": kinds["update"]["launches"]}
    for k in ("nystrom", "householder"):
        if ms_by.get(k, 0) > 0:
            roof_all[k] = {"bound": "fp64 latency (small dense algebra, reported separately, SURVEY 8d)",
                           "ms_per_step": ms_by[k]}
    # The dominant kernel: the three convolution classes are launches of ONE kernel template
    # (conv_tri_kernel / conv_tc_kernel<MODE>), the Gram class is several kernels; the template with
    # the largest summed time in the step wins, and of the convolution template its slowest
    # instantiation is the roofline object.  roofline_all keeps every class.
    tens = [k for k in roof_all if roof_all[k]["bound"] == "tensor"]
    convs = [k for k in ("conv_fwd", "scatter", "conv_els") if k in tens]
    conv_ms = sum(ms_by[k] for k in convs)
    if convs and conv_ms >= ms_by.get("gram", 0.0):
        dom = max(convs, key=lambda k: ms_by[k])
    else:
        dom = max(tens, key=lambda k: ms_by[k]) if tens else None
    roof = dict(roof_all[dom]) if dom else None
    if roof:
        top = max((k for k in roof_all if k in ms_by), key=lambda k: ms_by[k])
        roof.update({"kernel": dom,
                     "dominant_rule": ("kernel template with the largest summed time in the step "
                                       f"(convolution template {conv_ms:.2f} ms, Gram class "
                                       f"{ms_by.get('gram', 0.0):.2f} ms); its slowest instantiation"),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense 16-bit tensor rate) / 3: "
                                    "three fp16 MMA products per FP32-grade product",
                     "achieved_def": "algorithmic flops of the class in one step / its summed CUDA-event time "
                                     "(native profiler, one extra step on the launching stream)",
                     "traffic_def": "ncu dram read+write bytes per launch (profiles/r02_ncu_full.json)",
                     "achieved_note": "includes the operand split passes (amax + fp16 hi/lo split) inside each call",
                     "note": (f"the largest class overall is {top} ({roof_all[top]['bound']}"
                              + (f", frac {roof_all[top]['frac']:.3f}" if "frac" in roof_all[top] else "")
                              + "), see roofline_all") if top != dom else "also the largest class"})
    return roof, roof_all


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2004_08962_b200 import _native as nat

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nat.load()
    name = args.config
    dw = DeviceWorkload(name, world, rank, group)
    if name != "C3":
        _HOST_CACHE[(name, 1.0)] = dw.host[dw.slices[0]]  # the CPU sampler reuses the generated k-space
    stream = torch.cuda.current_stream()
    small = name != "C5"
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if small else None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        dw.step()
    torch.cuda.synchronize()
    dw.check()
    clocks = ClockSampler(local)
    times = []
    launches0 = nat.lib().hicu_launch_count()
    clocks.start()
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dw.step()
        e1.record(stream)
        barrier()
        times.append(e0.elapsed_time(e1))
    clock_info = clocks.stop()
    launches = nat.lib().hicu_launch_count() - launches0
    dw.check()
    # per-kernel-class CUDA-event times from one extra, untimed step
    kinds = None
    if dw.sharded is None:
        prof = nat.Profiler()
        barrier()
        dw.set_prof(prof)
        prof.reset()
        dw.step()
        barrier()
        dw.set_prof(None)
        kinds = prof.summary()
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    per_rank_units = _step_iterations(name) if name != "C3" else dw.spec.iterations * len(dw.slices)
    if name in ("C4", "C5") and world > 1 or name == "C5":
        units = per_rank_units * args.steps  # one volume: every rank works on the same iterations
    elif name == "C3":
        t = torch.tensor([per_rank_units * args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t)
        units = float(t.item())
    else:
        units = per_rank_units * args.steps * world
    value = units / (total_ms * 1e-3)

    # ---- end to end through the public API (host arrays in, host array out) ----
    e2e = None
    if not args.no_e2e:
        dw.e2e(group)  # warm-up (pinned pools, draw threads)
        reps = 1 if name in ("C5", "C3") else max(1, min(args.steps, 5))
        tot = 0.0
        its = 0
        h2d = d2h = 0
        for _ in range(reps):
            barrier()
            dt, n_it, h2d, d2h = dw.e2e(group)
            tot += dt
            its += n_it
        if world > 1:
            tt = torch.tensor([tot], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tot = float(tt.item())
            ii = torch.tensor([its], dtype=torch.float64, device="cuda")
            if name in ("C3",):
                dist.all_reduce(ii)
            elif name not in ("C4", "C5"):
                ii *= world
            its = float(ii.item())
        e2e = {"value": its / tot, "unit": "iters/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_call": 1e3 * tot / reps, "calls": reps, "iterations_per_call": its / reps,
               "path": {"C5": "sharded_reconstruct" if world > 1 else "hicu_reconstruct",
                        "C3": "reconstruct_slices"}.get(name, "hicu_reconstruct")
               + " from host numpy arrays (complex64 k-space, uint8 mask), result downloaded"}

    roof, roof_all, share, ms_by = None, None, None, None
    work = _work_per_step(dw)
    peaks = _load_json("MEASURED_PEAKS.json", {})
    if kinds is not None:
        roof, roof_all = roofline(kinds, work, peaks, profiled=(name == DEFAULT_CONFIG and world == 1))
        ms_by = {k: v["ms"] for k, v in kinds.items()}
        tot_ms = sum(ms_by.values())
        share = {k: (v / tot_ms if tot_ms > 0 else 0.0) for k, v in ms_by.items()}
    eff = None
    if world == 1:
        # dense-equivalent algorithmic flops (SURVEY 8d's F_iter) per second of the whole step
        flops = work["gram_dense_equiv"] + sum(work[k] for k in ("conv_fwd", "scatter", "conv_els"))
        eff = flops / (total_ms / args.steps * 1e-3) / 1e12

    # ---- CPU baseline: the reference package on a bounded sample, rank 0, N=1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = _host_threads()
        est_all, det_all = reference_sample(name, threads)
        est_one, det_one = reference_sample(name, 1)
        su = _step_iterations(name)
        cpu = {"value": su / est_all, "unit": "iters/s", "cores": threads, "kind": det_all["kind"],
               "sample": _sample_text(name, det_all), "cpu": _cpu_model(), "detail": det_all,
               "one_thread": {"value": su / est_one, "unit": "iters/s", "cores": 1, "detail": det_one}}

    if rank == 0:
        line = {
            "metric": "HICU iters/s", "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (world > 1 and name in ("C3", "C4", "C5")) else "weak", "vs_baseline": None,
            "dtype": "c64 (3xTF32 tcgen05 convs/Gram; fp64 reductions and nullspace)",
            "data": "synthetic (seeded phantoms with BASELINE.json shapes; paper_2004_08962_b200/synthetic.py)",
            "config": workload_config(name, world), "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches) // max(1, args.steps),
            "roofline": roof, "roofline_all": roof_all, "cpu_baseline": cpu, "clocks": clock_info,
            "kernel_share": share, "kernel_ms_per_step": ms_by,
            "kernel_ms_source": "one extra untimed step with the native CUDA-event profiler",
            "effective_tflops": eff,
            "step_ms": times,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
