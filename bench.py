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

value     device-timed whole-job cell updates/s, inputs resident in HBM
e2e       the same step through the public API from pinned HOST buffers
          (per-patch AoS, pipelined H2D / step / D2H), copies inside the timed region
roofline  fused kernel: algorithmic bytes 8*N*((p+2)^d + p^d) per patch ... / kernel time
cpu_baseline  the CPU oracle port (oracle/fv_oracle.c, OpenMP) on a bounded sample, rank 0, N=1

--impl reference times the reference algorithm's CPU port (the oracle; the
reference itself is pure Python and is not installed on the GPU box) on the
host cores and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
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
    ap.add_argument("--e2e-chunks", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--warmup-seconds", type=float, default=1.5,
                    help="keep warming up (beyond --warmup steps) until this much load time has "
                         "passed: B200 throttles for ~0.5 s after load onset (sw_power_cap "
                         "transient) before settling at full clock")
    return ap.parse_args()


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
            "sample": f"{sample} patches ({cells} cells) of the workload, {n} steps in {el:.1f} s, "
                      f"oracle/fv_oracle.c (literal run_sequential restatement, OpenMP over "
                      f"patches, gcc -O2 -ffp-contract=off)"}


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
                         "sample": f"{sample} patches per step of the workload (each step a bounded "
                                   f"sample), oracle/fv_oracle.c OpenMP"},
        "e2e": {"value": value, "unit": "cell updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    a = parse()
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
    from paper_2306_16731_b200.pipeline import StreamedStep

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

    t_w, warm = time.perf_counter(), 0
    while warm < max(3, a.warmup) or time.perf_counter() - t_w < a.warmup_seconds:
        step()
        warm += 1
        if warm % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(a.steps):
            ev[i][0].record(stream)
            _lib.check(lib.fvb_step(*args))
            ev[i][1].record(stream)
            if world > 1:
                dist.all_reduce(lam, op=dist.ReduceOp.MAX)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = start.elapsed_time(stop)
    kern_ms = statistics.mean(s.elapsed_time(e) for s, e in ev)
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

    # ---- e2e through the public API from pinned host buffers -------------
    e2e = None
    if not a.no_e2e:
        # Pinned host buffers: per rank N*((p+2)^d + p^d)*8 B per patch.  Bound
        # them to ~35% of the host's RAM shared by the ranks on this node, so an
        # 8-GPU run cannot exhaust host memory; larger shards time the e2e leg
        # on their first `ep` patches (reported as e2e.patches_per_gpu).
        nin, nout = shape.unknowns * shape.haloed_cells, shape.unknowns * shape.interior_cells
        try:
            host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        except (ValueError, OSError, AttributeError):
            host_ram = 64 << 30
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        ep = int(min(a.patches, 0.35 * host_ram / max(1, local_world) / (8 * (nin + nout))))
        ep = max(1, min(ep, int(os.environ.get("FVB_BENCH_E2E_MAX_PATCHES", ep))))
        eshape = fvb.BatchShape(a.dim, a.p, ep)
        # The device batches of the timed step are done with: free them so a
        # large shard (e.g. C5's 4 Mi patches on one GPU) has room for the
        # e2e staging buffers.
        del out
        if ep < a.patches:  # e2e on the shard's first ep patches: the same LCG stream
            del q
            torch.cuda.empty_cache()
            src = fvb.init_field_device(eshape, a.seed, patch_begin=rank * a.patches)
        else:
            src = q
        sdev = StreamedStep(eshape, chunks=a.e2e_chunks, flavour=flavour, device=dev)
        h_in = torch.empty(ep * nin, dtype=torch.float64, pin_memory=True)
        h_out = torch.empty(ep * nout, dtype=torch.float64, pin_memory=True)
        # host patches = the same field, per-patch AoS (ScatteredPatchSet order)
        aos = torch.empty(ep * nin, dtype=torch.float64, device=dev)
        _lib.check(lib.fvb_soa_to_aos(a.dim, a.p, ep, 1, src.data_ptr(), aos.data_ptr(), st))
        h_in.copy_(aos)
        del aos
        if ep < a.patches:  # the device path's eigenvalue of the same subset, for the check
            sub_out = torch.empty(ep * nout, dtype=torch.float64, device=dev)
            sub_lam = torch.zeros(1, dtype=torch.float64, device=dev)
            _lib.check(lib.fvb_step(flavour, a.dim, a.p, ep, src.data_ptr(), sub_out.data_ptr(),
                                    ctx.dt, ctx.h, ctx.params.gamma, 1, sub_lam.data_ptr(), None, st))
            if world > 1:
                dist.all_reduce(sub_lam, op=dist.ReduceOp.MAX)
            e2e_expect = float(sub_lam.item())
            del sub_out
        else:
            e2e_expect = reduced
        del src
        torch.cuda.empty_cache()
        elam = torch.zeros(1, dtype=torch.float64, device=dev)
        def e2e_step():
            slots = sdev.run(h_in, h_out, ctx)
            torch.amax(slots, dim=0, keepdim=True, out=elam)
            if world > 1:
                dist.all_reduce(elam, op=dist.ReduceOp.MAX)
            return float(elam.item())  # D2H read of the step's result
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.e2e_steps):
            r = e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        assert r == e2e_expect, f"e2e eigenvalue {r!r} != device path {e2e_expect!r}"
        hin, hout = sdev.bytes_per_step()
        e_cells = ep * a.p**a.dim * world
        # Context for e2e: the pinned host->device copy bandwidth of this box
        # (plain 2 GiB DMA), the bound the streamed step runs against.
        h2d_gbs = None
        try:
            nb = min(h_in.numel(), (2 << 30) // 8)
            tmp = torch.empty(nb, dtype=torch.float64, device=dev)
            cur = torch.cuda.current_stream(dev)
            tmp.copy_(h_in[:nb], non_blocking=True)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(cur)
            for _ in range(3):
                tmp.copy_(h_in[:nb], non_blocking=True)
            c1.record(cur)
            torch.cuda.synchronize()
            h2d_gbs = 3 * nb * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9
            del tmp
        except RuntimeError:
            h2d_gbs = None
        e_s = float(e_ms[0]) * 1e-3
        e2e = {"value": e_cells * a.e2e_steps / e_s,
               "unit": "cell updates/s", "h2d_bytes_per_step": hin, "d2h_bytes_per_step": hout,
               "path": f"public API StreamedStep: pinned host AoS -> H2D -> aos_to_soa -> "
                       f"fvb_step({a.flavour}) -> soa_to_aos -> D2H, {sdev.chunks} chunks on 3 "
                       f"streams, + eigenvalue read", "steps": a.e2e_steps,
               "patches_per_gpu": ep,
               "h2d_gbs_achieved": hin * a.e2e_steps / e_s / 1e9,
               "pcie_h2d_gbs_this_box": h2d_gbs}
        del sdev, h_in, h_out

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
                         "kernel": f"fvb {a.flavour} step (memset + kernel(s)), mean CUDA-event "
                                   f"time per launch {kern_ms:.4f} ms",
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "peak_source": peak_src,
                         "copy_gbs_this_box": copy_gbs},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": a.steps * launches_per_step,
            "clocks": clocks.summary(),
            "reduced_eigenvalue": reduced,
            "dt_next": dt_next,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
