"""Benchmark: cell updates/s of the batched 2D Euler FV step, 16x16 patches, fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--flavour fused|cascade|graph] [--patches T] [--dim 2] [--p 16]

Workload (BASELINE.json configs[2], the metric's config): 2D compressible
Euler, 16x16-cell patches + 1-cell halo, T = 2^20 patches per GPU (weak
scaling), one fp64 Rusanov step with the max-eigenvalue reduction, seeded
synthetic field (the reference's init_field LCG, generated in HBM).  Inputs
(10.9 GB) and outputs (8.6 GB) per GPU exceed the 126 MB L2, so no flush is
needed between steps.  A step = one fvb_step through the C ABI (fused
kernel) + at N>1 the NCCL all-reduce(max) of the eigenvalue (dt).

value       device-timed whole-job cell updates/s, inputs resident in HBM
exhaustive  the same with the exhaustive eigenvalue reduction (every cell's
            max_eigenvalue evaluated; the default filter skips provably
            smaller ones): value, ms_per_step, roofline frac
e2e         the same step through the reference's entry point run_launch
            (POOLED, SoA batch) from a pinned host ScatteredPatchSet: chunk
            DMA in -> permute -> step -> permute -> DMA out, pipelined over
            patch chunks on three streams, eigenvalue read back; every host
            byte crosses PCIe inside the timed region
roofline    fused kernel: algorithmic bytes 8*N*((p+2)^d + p^d) per patch / kernel time
extras      C4 (3D p=8, 100k patches) and C2 (2D p=3, 100k patches, L2
            flushed between steps) device-timed; task-graph build +
            instantiate vs replay at 1 / 64 patch chunks, beside the
            cascade it replaces (C2, C3 top point)
cpu_baseline  the CPU oracle port (oracle/fv_oracle.c, OpenMP) on a bounded sample, rank 0, N=1

--impl reference times the reference algorithm's CPU port (the oracle,
OpenMP C) on the host cores and prints the same JSON line with "impl":
"reference"; when the reference package itself is installed in
baseline/_ref (pip --target) its own run_batched /
run_sequential are timed beside it on a declared subset
("python_reference", subset-extrapolated per-cell rates).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cell updates/s (2D Euler, 16x16 patches, fp64) at 1/2/4/8 B200; % HBM peak"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--flavour", choices=["fused", "cascade", "graph"], default="fused")
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--patches", type=int, default=1 << 20, help="patches per GPU")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk-patches", type=int, default=0,
                    help="run_launch pipeline chunk (0: ~64 MB of input per chunk)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-exhaustive", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--warmup-seconds", type=float, default=1.5,
                    help="keep warming up (beyond --warmup steps) until this much load time has "
                         "passed: B200 throttles for ~0.5 s after load onset (sw_power_cap "
                         "transient) before settling at full clock")
    return ap.parse_args()


def ensure_world(a):
    """Honour --gpus: re-exec under torch.distributed.run when launched
    without it, refuse a WORLD_SIZE that disagrees."""
    env = os.environ.get("WORLD_SIZE")
    if env is None:
        if a.gpus > 1:
            port = 29500 + os.getpid() % 2000
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
                   f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        return
    if int(env) != a.gpus:
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={env}; launch N ranks with --gpus N")


def algo_bytes_per_patch(d: int, p: int) -> int:
    """Compulsory HBM bytes per patch: read (p+2)^d, write p^d cells x N doubles."""
    return 8 * (d + 2) * ((p + 2) ** d + p**d)


def hbm_peak():
    path = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def config_dict(a, world):
    return {
        "workload": f"{a.dim}D Euler, {a.p}x{a.p}{'x%d' % a.p if a.dim == 3 else ''} patches + 1-cell "
                    f"halo, {a.patches} patches per GPU, Rusanov fp64 step + max-eigenvalue reduce",
        "baseline_config": "BASELINE.json configs[2] (2D p16 patch-count sweep, top point 2^20)",
        "dim": a.dim, "patch_size": a.p, "patches_per_gpu": a.patches,
        "total_patches": a.patches * world, "flavour": a.flavour,
        "parallelism": f"patch shards x{world}, NCCL allreduce-max of lambda" if world > 1
        else "single GPU",
        "l2": "inputs+outputs per GPU >> 126 MB L2; no flush needed",
        "seed": a.seed, "dt": 1e-3, "h": 0.1, "gamma": 1.4,
    }


# ---------------------------------------------------------------------------
# clocks (nvml) sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int) -> None:
        self.samples, self.reasons = [], set()
        self.stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover
            self.err = str(exc)

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None),
                    "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU port (the oracle) timing: cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_cpu_port(a, seconds: float, min_steps: int = 1):
    from oracle import oracle  # the CPU port; only bench's baseline legs run it

    threads = oracle.default_threads()
    sample = max(64, min(a.patches, threads * 256))
    q = oracle.init_field_soa(a.dim, a.p, sample, a.seed)
    cells = sample * a.p**a.dim
    oracle.step_c(a.dim, a.p, sample, q, threads=threads)  # warm
    t0 = time.perf_counter()
    n = 0
    while n < min_steps or time.perf_counter() - t0 < seconds:
        oracle.step_c(a.dim, a.p, sample, q, threads=threads)
        n += 1
    el = time.perf_counter() - t0
    return {"value": n * cells / el, "unit": "cell updates/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{sample} patches ({cells} cells) of the workload, {n} steps in {el:.1f} s, "
                      f"oracle/fv_oracle.c (literal run_sequential restatement, OpenMP over "
                      f"patches, gcc -O2 -ffp-contract=off)"}


def time_python_reference(a, budget_s: float = 20.0):
    """The reference package itself (baseline/_ref, pip --target of
    /root/reference/pkg): run_batched (its fastest CPU realisation) with
    workers = cpu_count, SHARED, AoS, reduction on, on a declared subset,
    plus run_sequential on a smaller one.  Rates are per cell, so they
    extrapolate to the full workload (flat in T and workers).
    None when the package is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "patchbench").is_dir():
        return None
    sys.path.insert(0, str(ref))
    try:
        import numpy as np

        from oracle import oracle  # bit-identical init_field (LCG), fast
        from patchbench.bench import run_launch
        from patchbench.equations import EulerParameters
        from patchbench.executors import Realization, ReductionStrategy, WorkerPool
        from patchbench.kernelgraph import build_plan
        from patchbench.memory import DeviceArena, ScatteredPatchSet, TransferMode
        from patchbench.microkernels import TimeStepContext
        from patchbench.patchdata import BatchShape, Layout
    except Exception as exc:  # pragma: no cover
        return {"unavailable": f"import failed: {exc}"}
    finally:
        sys.path.remove(str(ref))
    workers = os.cpu_count() or 1
    ctx = TimeStepContext(1e-3, 0.1, EulerParameters(1.4))
    out = {"cpu_model": cpu_model(), "workers": workers, "kind": "reference (Python/numpy, "
           "baseline/_ref)", "label": "subset-extrapolated"}

    def launch_rate(real, t, samples):
        shape = BatchShape(a.dim, a.p, t)
        q = oracle.init_field_soa(a.dim, a.p, t, a.seed)
        aos = oracle.soa_to_aos_patches(q, a.dim, a.p, t, True).reshape(t, -1)
        nout = (a.dim + 2) * a.p**a.dim
        sc = ScatteredPatchSet(shape, [aos[i].copy() for i in range(t)],
                               [np.zeros(nout) for _ in range(t)])
        plan = build_plan(shape, True)
        with WorkerPool(workers) as pool:
            times = []
            for _ in range(samples + 1):  # the first is the warm-up
                r = run_launch(plan, sc, Layout.AOS, real, TransferMode.SHARED,
                               ReductionStrategy.GROUP_TREE, ctx, DeviceArena(), pool)
                times.append(r.total_s)
        mean = statistics.mean(times[1:])
        return {"value": t * a.p**a.dim / mean, "unit": "cell updates/s", "patches": t,
                "samples": samples, "mean_total_s": mean}

    t_batched = 4096 if a.dim == 2 and a.p >= 16 else (256 if a.dim == 3 else 10000)
    t0 = time.perf_counter()
    out["run_batched"] = launch_rate(Realization.BATCHED, min(t_batched, a.patches), 2)
    if time.perf_counter() - t0 < budget_s:
        out["run_sequential"] = launch_rate(Realization.SEQUENTIAL, min(8, a.patches), 1)
    return out


def run_reference(a, rank, world):
    if rank != 0:
        return
    from oracle import oracle

    threads = oracle.default_threads()
    # size one step at ~0.5 s of host work
    probe = max(16, threads * 16)
    q = oracle.init_field_soa(a.dim, a.p, probe, a.seed)
    t0 = time.perf_counter()
    oracle.step_c(a.dim, a.p, probe, q, threads=threads)
    per_patch = (time.perf_counter() - t0) / probe
    sample = int(max(probe, min(a.patches, 0.5 / max(per_patch, 1e-9))))
    q = oracle.init_field_soa(a.dim, a.p, sample, a.seed)
    for _ in range(a.warmup):
        oracle.step_c(a.dim, a.p, sample, q, threads=threads)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle.step_c(a.dim, a.p, sample, q, threads=threads)
    el = time.perf_counter() - t0
    cells = sample * a.p**a.dim
    value = a.steps * cells / el
    line = {
        "metric": METRIC, "value": value, "unit": "cell updates/s", "impl": "reference",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * el / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference init_field LCG)", "config": config_dict(a, world),
        "cpu_baseline": {"value": value, "unit": "cell updates/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} patches per step of the workload (each step a bounded "
                                   f"sample), oracle/fv_oracle.c OpenMP"},
        "e2e": {"value": value, "unit": "cell updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not a.no_extras:
        line["python_reference"] = time_python_reference(a)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def time_steps(step, stream, steps, world, dist, sync_every=8, warm_steps=3, warm_s=0.0):
    """Warm up (>= warm_steps and >= warm_s seconds of load), then time
    `steps` calls of step(): per-launch CUDA events around step() on
    `stream`, the whole region between barriers.  Returns (elapsed_ms,
    mean_launch_ms, warm_steps_done)."""
    import torch

    t_w, warm = time.perf_counter(), 0
    while warm < warm_steps or time.perf_counter() - t_w < warm_s:
        step()
        warm += 1
        if warm % sync_every == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(steps):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return start.elapsed_time(stop), statistics.mean(s.elapsed_time(e) for s, e in ev), warm


def device_config(fvb, lib, _lib, d, p, t, flush_l2, steps, dev, seed=0):
    """Device-timed fused step of one extra config (rank-local)."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    ctx = fvb.default_context()
    q = fvb.init_field_device(shape, seed)
    out = torch.empty(shape.output_size, dtype=torch.float64, device=dev)
    lam = torch.zeros(1, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    # L2 flush between steps: write 256 MB (> 126 MB L2), then read another
    # 256 MB so the L2 holds clean lines only -- the flush's dirty lines are
    # not written back inside the next timed step (measured: a write-only
    # flush costs C2 ~2 us of extra DRAM write-back)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if flush_l2 else None  # 256 MB > L2
    clean = torch.ones(64 << 20, dtype=torch.float32, device=dev) if flush_l2 else None
    times = []
    for i in range(steps + 3):
        if flush is not None:
            flush.fill_(float(i))
            clean.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(lib.fvb_step(_lib.FVB_FUSED, d, p, t, q.data_ptr(), out.data_ptr(), ctx.dt, ctx.h,
                                ctx.params.gamma, 1, lam.data_ptr(), None, st.cuda_stream))
        e1.record(st)
        if i >= 3:
            times.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in times)
    peak, _ = hbm_peak()
    gbs = t * algo_bytes_per_patch(d, p) / (ms * 1e-3) / 1e9
    return {"config": f"{d}D p={p} T={t}", "ms_per_step": ms, "value": t * p**d / (ms * 1e-3),
            "unit": "cell updates/s", "achieved_gbs": gbs, "frac": gbs / peak,
            "l2": "flushed between steps (256 MB write + 256 MB read: clean, cold L2)" if flush_l2
                  else "inputs > L2",
            "reduced_eigenvalue": float(lam.item())}


def graph_costs(fvb, d, p, t, dev, chunks=1):
    """Task-graph flavour: build + instantiate (first launch) vs replay."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    q = fvb.init_field_device(shape, 0)
    out = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64, device=dev), shape, False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    scratch = fvb.GpuScratch(shape, fvb.Realization.TASK_GRAPH, chunks=chunks)
    alloc_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    fvb.step_async(fvb.Realization.TASK_GRAPH, plan, q, out, ctx, scratch)  # builds + instantiates
    build_ms = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    first_ms = (time.perf_counter() - t0) * 1e3
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        fvb.step_async(fvb.Realization.TASK_GRAPH, plan, q, out, ctx, scratch)
    e1.record(st)
    torch.cuda.synchronize()
    res = {"config": f"{d}D p={p} T={t} chunks={chunks}", "scratch_alloc_ms": alloc_ms,
           "build_instantiate_ms": build_ms, "first_launch_ms": first_ms,
           "replay_ms": e0.elapsed_time(e1) / 10, "graph_nodes": scratch.graph_nodes()}
    scratch.close()
    if chunks == 1:  # the cascade on the same batch: what the graph replaces
        cs = fvb.GpuScratch(shape, fvb.Realization.BATCHED)
        fvb.step_async(fvb.Realization.BATCHED, plan, q, out, ctx, cs)
        e0.record(st)
        for _ in range(10):
            fvb.step_async(fvb.Realization.BATCHED, plan, q, out, ctx, cs)
        e1.record(st)
        torch.cuda.synchronize()
        res["cascade_ms"] = e0.elapsed_time(e1) / 10
        cs.close()
    return res


def main():
    a = parse()
    ensure_world(a)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2306_16731_b200 as fvb
    from paper_2306_16731_b200 import _lib

    # FVB_BENCH_DEVICE / FVB_BENCH_BACKEND: test scaffolding only -- run an
    # N-rank job on fewer GPUs (ranks share a device, gloo instead of NCCL) to
    # exercise the multi-rank path where one GPU is all there is
    local = int(os.environ.get("FVB_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("FVB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lib = fvb.load_library()
    flavour = {"fused": _lib.FVB_FUSED, "cascade": _lib.FVB_CASCADE, "graph": _lib.FVB_GRAPH}[a.flavour]
    realization = {"fused": fvb.Realization.PATCH_WISE, "cascade": fvb.Realization.BATCHED,
                   "graph": fvb.Realization.TASK_GRAPH}[a.flavour]
    shape = fvb.BatchShape(a.dim, a.p, a.patches)
    ctx = fvb.default_context()
    # this rank's shard of the global patch stream
    q = fvb.init_field_device(shape, a.seed, patch_begin=rank * a.patches)
    out = torch.empty(shape.output_size, dtype=torch.float64, device=dev)
    lam = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    st = stream.cuda_stream
    args = (flavour, a.dim, a.p, a.patches, q.data_ptr(), out.data_ptr(), ctx.dt, ctx.h,
            ctx.params.gamma, 1, lam.data_ptr(), None, st)

    def step():
        _lib.check(lib.fvb_step(*args))
        if world > 1:
            dist.all_reduce(lam, op=dist.ReduceOp.MAX)

    with ClockSampler(local) as clocks:
        elapsed_ms, kern_ms, warm = time_steps(step, stream, a.steps, world, dist,
                                               warm_steps=max(3, a.warmup), warm_s=a.warmup_seconds)
    t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, kern_ms = float(t[0]), float(t[1])
    reduced = float(lam.item())
    dt_next = fvb.admissible_dt(reduced, ctx.h)

    cells_per_step = a.patches * a.p**a.dim * world
    value = cells_per_step * a.steps / (elapsed_ms * 1e-3)
    bytes_launch = a.patches * algo_bytes_per_patch(a.dim, a.p)
    peak, peak_src = hbm_peak()
    achieved = bytes_launch / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{a.flavour}_d{a.dim}p{a.p}_T{a.patches}")
        except Exception:
            traffic = None
    launches_per_step = {"fused": 1, "cascade": 2 + 3 * a.dim, "graph": 2 + 3 * a.dim}[a.flavour]
    gpu_launches = a.steps * launches_per_step

    # ---- the exhaustive reduction (no eigenvalue filter) -------------------
    exhaustive = None
    if not a.no_exhaustive and a.flavour == "fused":
        lam_x = torch.zeros(1, dtype=torch.float64, device=dev)
        xargs = args[:10] + (lam_x.data_ptr(),) + args[11:]

        def xstep():
            _lib.check(lib.fvb_step(*xargs))
            if world > 1:
                dist.all_reduce(lam_x, op=dist.ReduceOp.MAX)

        with _lib.tuning(_lib.FVB_TUNE_REDUCE_FILTER, 0), ClockSampler(local) as xclocks:
            x_el, x_kern, _ = time_steps(xstep, stream, a.steps, world, dist, warm_steps=3,
                                         warm_s=a.warmup_seconds)
        xt = torch.tensor([x_el, x_kern], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(xt, op=dist.ReduceOp.MAX)
        x_el, x_kern = float(xt[0]), float(xt[1])
        x_ach = bytes_launch / (x_kern * 1e-3) / 1e9
        assert float(lam_x.item()) == reduced, "exhaustive and filtered reductions disagree"
        gpu_launches += a.steps
        exhaustive = {"value": cells_per_step * a.steps / (x_el * 1e-3), "unit": "cell updates/s",
                      "ms_per_step": x_el / a.steps, "roofline_frac": x_ach / peak,
                      "achieved_gbs": x_ach, "clocks": xclocks.summary(),
                      "what": "every finished cell's max_eigenvalue evaluated (FVB_TUNE_REDUCE_FILTER=0); "
                              "identical eigenvalue"}

    # ---- e2e through the reference entry point run_launch ------------------
    e2e = None
    if not a.no_e2e:
        # The host patch set: per rank N*((p+2)^d + p^d)*8 B per patch, pinned.
        # Bounded to ~35% of the host's RAM shared by the ranks on this node;
        # larger shards time the e2e leg on their first `ep` patches.
        nin, nout = shape.unknowns * shape.haloed_cells, shape.unknowns * shape.interior_cells
        try:
            host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        except (ValueError, OSError, AttributeError):
            host_ram = 64 << 30
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        ep = int(min(a.patches, 0.35 * host_ram / max(1, local_world) / (8 * (nin + nout))))
        ep = max(1, min(ep, int(os.environ.get("FVB_BENCH_E2E_MAX_PATCHES", ep))))
        eshape = fvb.BatchShape(a.dim, a.p, ep)
        del out, q
        torch.cuda.empty_cache()
        if ep < a.patches:  # the device path's eigenvalue of the same subset, for the check
            src = fvb.init_field_device(eshape, a.seed, patch_begin=rank * a.patches)
            sub_out = torch.empty(ep * nout, dtype=torch.float64, device=dev)
            sub_lam = torch.zeros(1, dtype=torch.float64, device=dev)
            _lib.check(lib.fvb_step(flavour, a.dim, a.p, ep, src.data_ptr(), sub_out.data_ptr(),
                                    ctx.dt, ctx.h, ctx.params.gamma, 1, sub_lam.data_ptr(), None, st))
            if world > 1:
                dist.all_reduce(sub_lam, op=dist.ReduceOp.MAX)
            e2e_expect = float(sub_lam.item())
            del src, sub_out
            torch.cuda.empty_cache()
        else:
            e2e_expect = reduced
        patches = fvb.init_field(eshape, a.seed, pinned=True, patch_begin=rank * a.patches)
        arena = fvb.DeviceArena(dev)
        eplan = fvb.build_plan(eshape, True)
        elam = torch.zeros(1, dtype=torch.float64, device=dev)

        def e2e_step():
            res = fvb.run_launch(eplan, patches, fvb.Layout.SOA, realization, fvb.TransferMode.POOLED,
                                 fvb.ReductionStrategy.GROUP_TREE, ctx, arena,
                                 chunk_patches=a.e2e_chunk_patches)
            r = res.reduced  # the step's result, read back to the host
            if world > 1:
                elam.fill_(r)
                dist.all_reduce(elam, op=dist.ReduceOp.MAX)
                r = float(elam.item())
            return r, res

        e2e_step()  # warm-up: pooled buffers, table upload path
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        splits = []
        e0.record(stream)
        for _ in range(a.e2e_steps):
            r, res = e2e_step()
            splits.append(res)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        assert r == e2e_expect, f"e2e eigenvalue {r!r} != device path {e2e_expect!r}"
        e_s = float(e_ms[0]) * 1e-3
        e_cells = ep * a.p**a.dim * world
        chunk = a.e2e_chunk_patches or max(1, (64 << 20) // (8 * nin))
        nchunks = -(-ep // chunk)
        # pinned blocks in patch order: chunks move by DMA (no pointer tables)
        hin = ep * nin * 8  # the patches
        hout = ep * nout * 8 + 8 * nchunks  # the outputs + the per-chunk eigenvalue slots
        # context: a plain pinned host->device DMA on this box
        h2d_gbs = duplex = None
        try:
            blk = torch.from_numpy(patches.in_block)
            nb = min(blk.numel(), (2 << 30) // 8)
            tmp = torch.empty(nb, dtype=torch.float64, device=dev)
            tmp.copy_(blk[:nb], non_blocking=True)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(3):
                tmp.copy_(blk[:nb], non_blocking=True)
            c1.record(stream)
            torch.cuda.synchronize()
            h2d_gbs = 3 * nb * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9
            # both directions at once in the step's H2D:D2H byte ratio (the
            # pipeline's steady state): the ceiling of the e2e leg
            no = int(nb * nout / nin)
            oblk = torch.from_numpy(patches.out_block)[:no]
            tmp_o = torch.empty(no, dtype=torch.float64, device=dev)
            s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            torch.cuda.synchronize()
            c0.record(stream)
            s_up.wait_stream(stream), s_dn.wait_stream(stream)
            for _ in range(3):
                with torch.cuda.stream(s_up):
                    tmp.copy_(blk[:nb], non_blocking=True)
                with torch.cuda.stream(s_dn):
                    oblk.copy_(tmp_o, non_blocking=True)
            stream.wait_stream(s_up), stream.wait_stream(s_dn)
            c1.record(stream)
            torch.cuda.synchronize()
            dup_s = c0.elapsed_time(c1) * 1e-3 / 3
            duplex = {"h2d_gbs": nb * 8 / dup_s / 1e9, "d2h_gbs": no * 8 / dup_s / 1e9,
                      "step_bound_cells_per_s": nb / nin * a.p**a.dim / dup_s * world}
            del tmp, tmp_o
        except RuntimeError:
            h2d_gbs = None
        e2e = {"value": e_cells * a.e2e_steps / e_s,
               "unit": "cell updates/s", "h2d_bytes_per_step": hin, "d2h_bytes_per_step": hout,
               "path": f"run_launch(POOLED, SoA, {realization.value}) on a pinned host "
                       f"ScatteredPatchSet ({ep} per-patch AoS arrays in one pinned block): per chunk "
                       f"H2D DMA -> device AoS->SoA permutation -> {a.flavour} step -> SoA->AoS -> "
                       f"D2H DMA, {nchunks} chunks pipelined on 3 streams (fvb_launch_table), "
                       f"eigenvalue read back",
               "steps": a.e2e_steps, "patches_per_gpu": ep,
               "mean_split_s": {k: statistics.mean(getattr(s, k) for s in splits)
                                for k in ("total_s", "compute_s", "transfer_s", "alloc_s")},
               "h2d_gbs_achieved": hin * a.e2e_steps / e_s / 1e9,
               "pcie_h2d_gbs_this_box": h2d_gbs,
               "pcie_duplex_this_box": duplex}
        gpu_launches += (a.e2e_steps) * 3 * nchunks  # permute-in + step + permute-out per chunk
        del patches, arena
        torch.cuda.empty_cache()

    # ---- extra configs (rank-local, device-timed) --------------------------
    extras = None
    if not a.no_extras and rank == 0 and world == 1:
        extras = {"C4": device_config(fvb, lib, _lib, 3, 8, 100_000, False, 50, dev),
                  "C2": device_config(fvb, lib, _lib, 2, 3, 100_000, True, 50, dev),
                  "task_graph": [graph_costs(fvb, d_, p_, t_, dev, chunks=c)
                                 for d_, p_, t_ in ((2, 3, 100_000), (2, 16, 1 << 20))
                                 for c in (1, 64)]}  # 4096 chunks: profiles/r02_task_graph.csv
        gpu_launches += 2 * 53 + 2 * (11 * (1 + 64) + 11) * (2 + 3 * 2)
        torch.cuda.empty_cache()

    # Context for the roofline: a plain device-to-device copy measured on this
    # box in this run (the kind of operation MEASURED_PEAKS' hbm_gbs is).
    copy_gbs = None
    try:
        nbytes = 4 << 30
        src_b = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
        dst_b = torch.empty_like(src_b)
        for _ in range(3):
            dst_b.copy_(src_b)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(10):
            dst_b.copy_(src_b)
        c1.record(stream)
        torch.cuda.synchronize()
        copy_gbs = 2 * nbytes * 10 / (c0.elapsed_time(c1) * 1e-3) / 1e9
        del src_b, dst_b
    except RuntimeError:
        pass

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = time_cpu_port(a, a.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell updates/s", "n_gpus": world,
            "steps": a.steps, "warmup": max(3, a.warmup), "ms_per_step": elapsed_ms / a.steps,
            "warmup_done": {"steps": warm, "min_seconds": a.warmup_seconds,
                            "why": "steady-state clocks: ~0.5 s sw_power_cap transient at load onset"},
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference init_field LCG, generated in HBM)",
            "config": config_dict(a, world),
            "hbm_frac": achieved / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"fvb {a.flavour} step ({'one kernel, no memset' if a.flavour == 'fused' else 'stage kernels'}), mean CUDA-event "
                                   f"time per launch {kern_ms:.4f} ms",
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "peak_source": peak_src,
                         "copy_gbs_this_box": copy_gbs},
            "exhaustive": exhaustive,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "extras": extras,
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
            "reduced_eigenvalue": reduced,
            "dt_next": dt_next,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
