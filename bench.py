"""HICU B200 benchmark (driver contract: one JSON line on rank 0).

Workload = BASELINE.json configs[1] ("C2"): 256x256 k-space, 16 coils
SVD-compressed to 8 on the device, 1D variable-density phase-encode mask R=4,
5x5x8 kernel (n = 200), rank 60, center-out schedule 64^2 -> 128^2 -> full
with 25/25/50 outer iterations, p = 8, G = 5 gradient steps per iteration.
A step is one full reconstruction (100 outer iterations) of one synthetic
slice; metric = HICU outer iterations per second.

* ``value``: device-resident (16-coil k-space, mask and all host-seeded
  sketch/JL draws already in HBM); CUDA events around each step on the
  compute stream; L2 flushed between steps (256 MiB write, untimed).
* ``e2e``: the public API ``hicu_reconstruct`` from host numpy arrays
  (draws made on host worker threads, uploaded, result downloaded).
* ``roofline``: the dominant tensor-core kernel class (Gram or one of the
  three convolutions) from the native CUDA-event profiler over the timed
  region, against the measured TF32 peak / 3 (3xTF32); ``roofline_all``
  lists every class, including the HBM-bound update and the fp64 nullspace
  (latency-bound, reported separately as SURVEY §8d asks).
* ``batched`` (supplementary, N=1): 8 independent C2 slices reconstructed 4
  at a time on concurrent CUDA streams (``hicu_reconstruct_batch``, the
  multi-slice C3 path); ``value`` stays the single-slice C2 metric.
* ``cpu_baseline``: the oracle port (numpy/scipy restatement of the
  reference) on a bounded sample (coil compression + one outer iteration per
  stage), extrapolated to the schedule; rank 0, N=1 only.
* ``--impl reference``: the same oracle port as the reference arm (the
  reference is pure Python and cannot be shipped to the GPU box; its port is
  pinned to the reference's golden vectors in tests/).

N > 1 (torchrun): replicas — each rank reconstructs its own slice (no data-
path collective); value = all ranks' iterations / max-over-ranks time.
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

CONFIG = "C2"


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


def workload_config(spec):
    return {
        "workload": (f"{spec.name} (BASELINE.json configs[1]): 256x256, {spec.coils_in}->{spec.coils_out} coils "
                     "(device SVD coil compression), 1D VD phase-encode mask R=4, SNR 30 dB, kernel 5x5x8 (n=200), "
                     f"rank {spec.rank}, stages 64^2/128^2/full x 25/25/50 iterations, p=8, G=5"),
        "iterations_per_step": spec.iterations,
        "kernel": list(spec.kernel),
        "rank": spec.rank,
        "stages": [[s[0], s[1], s[2], s[3]] for s in spec.stages],
        "l2": "flushed between steps (256 MiB device write, untimed)",
        "parallelism": "replicas (one slice per GPU, no collective)",
    }


# ---------------------------------------------------------------------------
# CPU (oracle port) legs
# ---------------------------------------------------------------------------


def oracle_sample(x0, mask, spec, threads: int):
    """Coil compression + one outer iteration of each stage with the oracle
    port; returns (estimated seconds for the full schedule, details)."""
    from threadpoolctl import threadpool_limits

    from oracle import hicu_oracle as O

    with threadpool_limits(threads):
        t = time.perf_counter()
        xc, mc, _ = O.coil_compress(x0, mask, spec.coils_out)
        t_cc = time.perf_counter() - t
        per = []
        for si, (region, p, G, iters) in enumerate(spec.stages):
            t = time.perf_counter()
            O.hicu_reconstruct(xc, mc, spec.kernel, [(region, p, G, 1)], spec.rank, seed=si)
            per.append(time.perf_counter() - t)
    est = t_cc + sum(st[3] * t_it for st, t_it in zip(spec.stages, per))
    return est, {"coil_s": t_cc, "iter_s_by_stage": per}


def run_reference(args):
    """Reference arm: the oracle port of the reference's CPU path, all host
    threads, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2004_08962_b200.synthetic import CONFIGS, make_config

    spec = CONFIGS[CONFIG]
    ksp, mask, x0 = make_config(CONFIG)
    threads = _host_threads()
    for _ in range(args.warmup):
        oracle_sample(x0, mask, spec, threads)
    est_total = 0.0
    samples = []
    for _ in range(args.steps):
        est, det = oracle_sample(x0, mask, spec, threads)
        est_total += est
        samples.append(det)
    value = spec.iterations * args.steps / est_total
    line = {
        "metric": "HICU iters/s", "value": value, "unit": "iters/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * est_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": workload_config(spec), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": "coil compression + 1 outer iteration per stage, extrapolated to 25/25/50",
                         "cpu": _cpu_model(), "last_sample": samples[-1]},
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


def _flops_by_kind(spec, n, ell, regions, ccfg):
    """Algorithmic work per launch group, per stage."""
    out = []
    for st, reg in zip(spec.stages, regions):
        s = reg.s
        p = st[1]
        out.append({
            "gram": 4.0 * s * n * (n + 1),                      # Hermitian H^H H, real flops
            "conv_fwd": 8.0 * s * n * p,                        # u = H(y) Q~
            "scatter": 8.0 * s * n * p,                         # g = col2im(Q~^H u)
            "conv_els": 8.0 * s * n * p,                        # w = H(g) Q~ (+ <w,u>, |w|^2)
            "update_bytes": 25.0 * ccfg["N"],                   # y, g read, y write, mask
            "iters": st[3],
            "G": st[2],
        })
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2004_08962_b200 as H
    from paper_2004_08962_b200 import _native as nat
    from paper_2004_08962_b200.coil import coil_compress_device
    from paper_2004_08962_b200.hankel import to_dev
    from paper_2004_08962_b200.solver import ReconEngine, draw_stage
    from paper_2004_08962_b200.synthetic import CONFIGS, make_config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nat.load()
    spec = CONFIGS[CONFIG]
    ksp, mask, x0 = make_config(CONFIG, slice_index=rank)
    kernel = H.KernelMask.full(spec.kernel)
    sched = H.SolverSchedule(rank=spec.rank, stages=[H.StageSpec(*s) for s in spec.stages], seed=rank)
    nc, nv = spec.coils_in, spec.coils_out
    dims_c = x0.shape[:-1] + (nv,)
    regions = sched.validate(kernel, dims_c)
    n = kernel.n
    ell = math.ceil(1.5 * spec.rank)

    # ---- device-resident inputs ----
    xd16 = to_dev(x0).reshape(-1)
    md16 = to_dev(mask, np.uint8).reshape(-1)
    ydev, mdev, _, _ = coil_compress_device(xd16, md16, nc, nv)
    eng = ReconEngine(ydev, mdev, dims_c, kernel, sched, regions)
    for si, st in enumerate(sched.stages):
        om, pb = draw_stage(sched, si, st, n)
        eng.set_host_draws(si, om, pb)
    prof = nat.Profiler()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def one_step():
        y, _, _, _ = coil_compress_device(xd16, md16, nc, nv)
        eng.y.copy_(y)
        eng.status.zero_()
        eng.run_all()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    eng.check_status()
    clocks = ClockSampler(local)
    times = []
    launches0 = nat.lib().hicu_launch_count()
    clocks.start()
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_step()
        e1.record(stream)
        barrier()
        times.append(e0.elapsed_time(e1))
    clock_info = clocks.stop()
    launches = nat.lib().hicu_launch_count() - launches0
    eng.check_status()
    # per-kernel-class CUDA-event times from one extra, untimed step (the
    # event records between kernels would perturb the timed steps)
    flush.fill_(1.0)
    barrier()
    eng.prof = prof
    prof.reset()
    one_step()
    barrier()
    eng.prof = None
    kinds = prof.summary()
    eng.check_status()
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    iters_all = spec.iterations * args.steps * world
    value = iters_all / (total_ms * 1e-3)

    # ---- end to end through the public API (host arrays in, host array out) ----
    e2e = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup // 2)):
            H.hicu_reconstruct(x0, mask, kernel, sched, tail_energy_threshold=0, coil_compress=nv)
        e2e_t = []
        rep = None
        for _ in range(args.steps):
            barrier()
            t = time.perf_counter()
            _, rep = H.hicu_reconstruct(x0, mask, kernel, sched, tail_energy_threshold=0, coil_compress=nv)
            e2e_t.append(time.perf_counter() - t)
        tot = sum(e2e_t)
        if world > 1:
            tt = torch.tensor([tot], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tot = float(tt.item())
        e2e = {"value": spec.iterations * args.steps * world / tot, "unit": "iters/s",
               "h2d_bytes_per_step": rep.device["h2d_bytes"], "d2h_bytes_per_step": rep.device["d2h_bytes"],
               "ms_per_step": 1e3 * tot / args.steps,
               "path": "paper_2004_08962_b200.hicu_reconstruct(numpy c64 x0, mask, coil_compress=8)"}

    # ---- supplementary: independent slices on concurrent streams (C3-style batching) ----
    batched = None
    if world == 1 and not args.no_e2e:
        nb_slices, conc = 8, 4
        data = [make_config(CONFIG, slice_index=i) for i in range(nb_slices)]
        bx, bm = [d[2] for d in data], [d[1] for d in data]
        H.hicu_reconstruct_batch(bx, bm, kernel, sched, concurrency=conc, tail_energy_threshold=0, coil_compress=nv)
        dt = float("inf")
        for _ in range(2):  # best of two
            torch.cuda.synchronize()
            t = time.perf_counter()
            H.hicu_reconstruct_batch(bx, bm, kernel, sched, concurrency=conc, tail_energy_threshold=0,
                                     coil_compress=nv)
            torch.cuda.synchronize()
            dt = min(dt, time.perf_counter() - t)
        batched = {"value": nb_slices * spec.iterations / dt, "unit": "iters/s", "slices": nb_slices,
                   "concurrency": conc, "ms_per_slice": 1e3 * dt / nb_slices,
                   "path": "hicu_reconstruct_batch: independent C2 slices on concurrent CUDA streams, host arrays",
                   "timing": "wall clock between device-wide synchronizations, best of 2 after a warm-up batch"}

    # ---- roofline of the dominant kernel class ----
    ccfg = {"N": int(np.prod(dims_c))}
    work = _flops_by_kind(spec, n, ell, regions, ccfg)
    flops_total = {k: 0.0 for k in ("gram", "conv_fwd", "scatter", "conv_els")}
    launches_expected = {k: 0 for k in flops_total}
    for w in work:
        for k in flops_total:
            per_launch_groups = w["iters"] * (1 if k == "gram" else w["G"])
            flops_total[k] += w[k] * per_launch_groups  # the profiled step
            launches_expected[k] += per_launch_groups
    ms_by = {k: v["ms"] for k, v in kinds.items()}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    tf32 = json.load(open(os.path.join(ROOT, "profiles", "tf32_peak_r01.json")))
    hbm = peaks.get("hbm_gbs", 6650.0)
    # ncu --set full captures of full-stage launches (scripts/ncu_full.sh -> profiles/r01_ncu_full_v16.json)
    ncu_by = {}
    try:
        for rec in json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_full_v16.json"))):
            ncu_by[rec["kernel"]] = rec
    except (OSError, ValueError):
        pass
    ncu_name = {"gram": "gram_tc_kernel", "conv_fwd": "void conv_tc_kernel<0, 0>", "scatter": "void conv_tc_kernel<2, 0>",
                "conv_els": "void conv_tc_kernel<1, 0>", "update": "update_kernel"}

    def traffic(kind):
        rec = ncu_by.get(ncu_name.get(kind, ""))
        if not rec or rec.get("dram_read_bytes") is None:
            return None
        return rec["dram_read_bytes"] + (rec.get("dram_write_bytes") or 0.0)

    tf32_peak = tf32["tf32_tflops"] / 3.0
    roof_all = {}
    for k in ("gram", "conv_fwd", "scatter", "conv_els"):
        if k not in ms_by or ms_by[k] <= 0:
            continue
        nl = max(1, kinds[k]["launches"])
        ach = flops_total[k] / (ms_by[k] * 1e-3) / 1e12
        roof_all[k] = {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s",
                       "frac": ach / tf32_peak, "traffic": traffic(k), "launches": nl,
                       "avg_launch_ms": ms_by[k] / nl, "flops_per_launch_avg": flops_total[k] / nl}
    if "update" in ms_by and ms_by["update"] > 0:
        bytes_total = sum(w["update_bytes"] * w["iters"] * w["G"] for w in work)
        ach = bytes_total / (ms_by["update"] * 1e-3) / 1e9
        roof_all["update"] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                              "traffic": traffic("update"), "launches": kinds["update"]["launches"]}
    for k in ("nystrom", "householder"):
        if k in ms_by:
            roof_all[k] = {"bound": "fp64 latency (single-CTA small dense algebra, reported separately, SURVEY 8d)",
                           "ms_per_step": ms_by[k],
                           "us_per_iteration": 1e3 * ms_by[k] / spec.iterations}
    # the roofline object: the dominant tensor-core kernel class (K1 Gram / K4-K6 convolutions)
    dom = max((k for k in roof_all if roof_all[k]["bound"] == "tensor"), key=lambda k: ms_by[k])
    roof = dict(roof_all[dom])
    roof.update({"kernel": dom, "peak_source": "measured TF32 dense (profiles/tf32_peak_r01.json) / 3 for 3xTF32",
                 "achieved_def": "algorithmic flops of all launches of the class / their summed CUDA-event time",
                 "traffic_def": "ncu dram read+write bytes of one full-stage launch (profiles/r01_ncu_full_v16.json)"})
    share = {k: (v / sum(ms_by.values()) if sum(ms_by.values()) > 0 else 0.0) for k, v in ms_by.items()}
    grad_tflops = sum(flops_total.values()) / (total_ms / args.steps * 1e-3) / 1e12 if world == 1 else None

    # ---- CPU baseline (oracle port), rank 0, N=1 only ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = _host_threads()
        est, det = oracle_sample(x0, mask, spec, threads)
        cpu = {"value": spec.iterations / est, "unit": "iters/s", "cores": threads, "kind": "port",
               "sample": "coil compression + 1 outer iteration per stage of C2, extrapolated to 25/25/50",
               "cpu": _cpu_model(), "detail": det}

    if rank == 0:
        line = {
            "metric": "HICU iters/s", "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64 (3xTF32 tcgen05 convs/Gram; fp64 reductions and nullspace)",
            "data": "synthetic", "config": workload_config(spec), "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches) // max(1, args.steps),
            "roofline": roof, "roofline_all": roof_all, "cpu_baseline": cpu, "clocks": clock_info,
            "batched": batched,
            "kernel_share": share, "kernel_ms_per_step": dict(ms_by),
            "kernel_ms_source": "one extra untimed step with the native CUDA-event profiler",
            "gram_grad_tflops": grad_tflops,
            "step_ms": times,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
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
