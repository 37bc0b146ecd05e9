"""Patch-update entry point and synthetic fields (the reference's bench.py API).

``run_launch`` keeps the signature and result type of
pkg/src/patchbench/bench.py:209-259 -- acquire, gather, compute, scatter,
release, with the same timing split -- and routes the compute step to a GPU
realisation.  ``init_field`` generates the reference's seeded field
(bench.py:107-133) directly in HBM with the jump-ahead LCG kernel
(bit-identical, including sharded generation for multi-GPU runs).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from . import _lib
from .context import TimeStepContext
from .equations import EulerParameters
from .executors import (ExecutionTrace, Realization, ReductionStrategy, run_batched,
                        run_patchwise, run_taskgraph)
from .kernelgraph import KernelPlan
from .memory import (DeviceArena, DevicePatchSet, ScatteredPatchSet, TransferMode,
                     acquire_buffers, allocate_scattered, gather_patches, release_buffers,
                     scatter_results)
from .patchdata import BatchShape, DeviceFieldView, Layout

__all__ = ["LaunchResult", "run_launch", "init_field", "init_field_device", "admissible_dt"]


@dataclass
class LaunchResult:
    total_s: float
    compute_s: float
    transfer_s: float
    alloc_s: float
    reduced: float | None
    trace: ExecutionTrace | None


def init_field_device(shape: BatchShape, seed: int, gamma: float = 1.4, device="cuda",
                      patch_begin: int = 0, out=None) -> DeviceFieldView:
    """Haloed SoA input in HBM holding init_field's bits for patches
    [patch_begin, patch_begin + T) of the seed's global patch stream."""
    import torch

    if out is None:
        out = torch.empty(shape.input_size, dtype=torch.float64, device=device)
    _lib.check(_lib.load().fvb_init_field(shape.dim, shape.patch_size, shape.patch_count,
                                          patch_begin, seed & ((1 << 64) - 1), gamma,
                                          out.data_ptr(),
                                          torch.cuda.current_stream(out.device).cuda_stream))
    return DeviceFieldView(out, shape, True)


def init_field(shape: BatchShape, seed: int, gamma: float = 1.4,
               pinned: bool = True) -> ScatteredPatchSet:
    """Seeded admissible field on a fresh scattered (host, AoS) patch set,
    like the reference's init_field; generated on the GPU, copied back."""
    import torch

    q = init_field_device(shape, seed, gamma)
    aos = torch.empty_like(q.tensor)
    _lib.check(_lib.load().fvb_soa_to_aos(shape.dim, shape.patch_size, shape.patch_count, 1,
                                          q.data_ptr(), aos.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    sc = allocate_scattered(shape, pinned=pinned)
    torch.from_numpy(sc.in_block).copy_(aos)
    return sc


def admissible_dt(reduced: float, h: float, cfl: float = 0.5) -> float:
    """dt = cfl*h/lambda (builder addition; the reference stops at lambda,
    SPEC.md:8).  Computed by the library's host function so every rank and
    the CPU oracle evaluate the identical IEEE expression."""
    return float(_lib.load().fvb_admissible_dt(reduced, h, cfl))


_EXECUTORS = {
    Realization.PATCH_WISE: lambda plan, b, s, ctx, pool, strat, wl: run_patchwise(
        plan, b.input_view, b.output_view, s, ctx, pool, strat, wl),
    Realization.BATCHED: lambda plan, b, s, ctx, pool, strat, wl: run_batched(
        plan, b.input_view, b.output_view, s, ctx, pool, strat),
    Realization.TASK_GRAPH: lambda plan, b, s, ctx, pool, strat, wl: run_taskgraph(
        plan, b.input_view, b.output_view, s, ctx, pool, strat),
}


def run_launch(plan: KernelPlan, scattered, layout: Layout, realization: Realization,
               transfer_mode: TransferMode, strategy: ReductionStrategy, ctx: TimeStepContext,
               arena: DeviceArena, pool=None, workgroup_limit: int = 1024,
               scratch=None) -> LaunchResult:
    """One full launch: acquire, gather, compute, scatter, release.

    ``layout`` is the reference's batch layout (patchdata.py:49-58): the
    device batch is gathered into it (AoS: a straight DMA of the host
    patches; SoA / AoSoA: DMA + one permutation kernel) and the kernels run
    on it natively (SoA is the fastest on B200, profiles/r01_layouts.csv).
    In SHARED mode the DevicePatchSet's own layout is used.  ``scratch``
    optionally passes a GpuScratch (plan-owned arena / instantiated graph).
    """
    import torch

    if realization not in _EXECUTORS:
        raise ValueError(f"{realization.value} is the CPU golden run, not a GPU realisation")
    sync = torch.cuda.synchronize
    sync()
    t_start = time.perf_counter()
    t0 = time.perf_counter()
    buffers = acquire_buffers(plan.shape, transfer_mode, arena, scattered, layout)
    alloc_s = time.perf_counter() - t0
    transfer_s = 0.0
    if transfer_mode is not TransferMode.SHARED:
        t0 = time.perf_counter()
        gather_patches(scattered, buffers)
        sync()
        transfer_s += time.perf_counter() - t0
    t0 = time.perf_counter()
    reduced, trace = _EXECUTORS[realization](plan, buffers, scratch, ctx, pool, strategy,
                                             workgroup_limit)
    sync()
    compute_s = time.perf_counter() - t0
    if transfer_mode is not TransferMode.SHARED:
        t0 = time.perf_counter()
        scatter_results(buffers, scattered)
        sync()
        transfer_s += time.perf_counter() - t0
    t0 = time.perf_counter()
    release_buffers(buffers, arena)
    alloc_s += time.perf_counter() - t0
    total_s = time.perf_counter() - t_start
    return LaunchResult(total_s, compute_s, transfer_s, alloc_s, reduced, trace)


def default_context(gamma: float = 1.4, dt: float = 1e-3, h: float = 0.1,
                    check: bool = False) -> TimeStepContext:
    """The reference benchmark's run parameters (bench.py:150-153)."""
    return TimeStepContext(dt, h, EulerParameters(gamma), check)
