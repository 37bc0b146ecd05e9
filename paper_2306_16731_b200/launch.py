"""Patch-update entry point and synthetic fields (the reference's bench.py API).

``run_launch`` keeps the signature and result type of
pkg/src/patchbench/bench.py:209-259 -- acquire, gather, compute, scatter,
release, with the same timing split -- and routes the compute step to a GPU
realisation.  ``init_field`` generates the reference's seeded field
(bench.py:107-133) directly in HBM with the jump-ahead LCG kernel
(bit-identical, including sharded generation for multi-GPU runs).
"""

from __future__ import annotations

import contextlib
import ctypes
import time

import numpy as np
from dataclasses import dataclass

from . import _lib
from .context import TimeStepContext
from .equations import EulerParameters
from .errors import WorkgroupLimitError
from .executors import (ExecutionTrace, Realization, ReductionStrategy, run_batched,
                        run_patchwise, run_taskgraph)
from .kernelgraph import KernelPlan
from .memory import (DeviceArena, DevicePatchSet, ScatteredPatchSet, TransferMode,
                     acquire_buffers, allocate_scattered, gather_patches, release_buffers,
                     scatter_results)
from .patchdata import LAYOUT_CODES, BatchShape, DeviceFieldView, Layout

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


def init_field(shape: BatchShape, seed: int, gamma: float = 1.4, pinned: bool = True,
               patch_begin: int = 0) -> ScatteredPatchSet:
    """Seeded admissible field on a fresh scattered (host, AoS) patch set,
    like the reference's init_field (bench.py:107-133); generated on the GPU
    (jump-ahead LCG), copied back.  pinned=True: views into pinned blocks
    (device-addressable); pinned=False: T independently allocated arrays,
    like the reference's allocate_scattered."""
    import torch

    q = init_field_device(shape, seed, gamma, patch_begin=patch_begin)
    aos = torch.empty_like(q.tensor)
    _lib.check(_lib.load().fvb_soa_to_aos(shape.dim, shape.patch_size, shape.patch_count, 1,
                                          q.data_ptr(), aos.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    del q
    if pinned:
        sc = allocate_scattered(shape, pinned=True, zero=False)
        torch.from_numpy(sc.in_block).copy_(aos)
        sc.out_block[:] = 0.0
        return sc
    host = aos.cpu().numpy()
    nin, nout = shape.unknowns * shape.haloed_cells, shape.unknowns * shape.interior_cells
    return ScatteredPatchSet(shape, [host[i * nin:(i + 1) * nin].copy() for i in range(shape.patch_count)],
                             [np.zeros(nout) for _ in range(shape.patch_count)])


def admissible_dt(reduced: float, h: float, cfl: float = 0.5) -> float:
    """dt = cfl*h/lambda (builder addition; the reference stops at lambda,
    SPEC.md:8).  Computed by the library's host function so every rank and
    the CPU oracle evaluate the identical IEEE expression."""
    return float(_lib.load().fvb_admissible_dt(reduced, h, cfl))


_EXECUTORS = {
    Realization.PATCH_WISE: lambda plan, b, ctx, pool, strat, wl: run_patchwise(
        plan, b.input_view, b.output_view, b.scratch, ctx, pool, strat, wl),
    Realization.BATCHED: lambda plan, b, ctx, pool, strat, wl: run_batched(
        plan, b.input_view, b.output_view, b.scratch, ctx, pool, strat),
    Realization.TASK_GRAPH: lambda plan, b, ctx, pool, strat, wl: run_taskgraph(
        plan, b.input_view, b.output_view, b.scratch, ctx, pool, strat),
}


def run_launch(plan: KernelPlan, scattered, layout: Layout, realization: Realization,
               transfer_mode: TransferMode, strategy: ReductionStrategy, ctx: TimeStepContext,
               arena: DeviceArena, pool=None, workgroup_limit: int = 1024,
               chunk_patches: int = 0) -> LaunchResult:
    """One full launch: acquire, gather, compute, scatter, release
    (bench.py:209-259), same signature and result.

    ``scattered`` is a ScatteredPatchSet of T per-patch host AoS arrays
    (pinned blocks, or independently allocated arrays registered for this
    launch only, see memory.py), or a DevicePatchSet already in HBM.

    * SHARED: the step runs in place on the per-patch arrays through pointer
      tables (no batch buffers, transfer_s = 0.0).
    * EXPLICIT_COPY / POOLED: arena batch buffers in ``layout``; gather,
      step, scatter pipelined over patch chunks of ``chunk_patches`` (0:
      ~64 MB of input each) on three streams (fvb_launch_table) -- PCIe
      reads, compute and PCIe writes of different chunks overlap.  Pinned
      blocks move by chunk DMA, independently allocated arrays by a host
      gather into pinned chunks + DMA (no registration).  compute_s is the
      step kernels' device time, transfer_s the rest of the launch.

    The reduced eigenvalue and the outputs are bit-identical for every mode,
    layout, chunking and realisation (patches are independent; max is exact).
    """
    import torch

    from .executors import FLAVOUR_OF, _admissible, _plan_handle, gpu_kernel_launches, trace_of
    from .memory import DevicePatchSet

    if realization not in _EXECUTORS:
        raise ValueError(f"{realization.value} is the CPU golden run, not a GPU realisation")
    if realization is Realization.PATCH_WISE and plan.shape.haloed_cells > workgroup_limit:
        raise WorkgroupLimitError(
            f"(p+2)^d = {plan.shape.haloed_cells} exceeds workgroup limit {workgroup_limit}; "
            "the patch must be broken down manually")
    sync = torch.cuda.synchronize
    sync()
    t_start = time.perf_counter()
    t0 = time.perf_counter()
    buffers = acquire_buffers(plan.shape, layout, transfer_mode, arena, scattered)
    alloc_s = time.perf_counter() - t0
    if isinstance(scattered, DevicePatchSet):  # resident batch: the executor alone
        t0 = time.perf_counter()
        reduced, trace = _EXECUTORS[realization](plan, buffers, ctx, pool, strategy, workgroup_limit)
        sync()
        compute_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        release_buffers(buffers, arena)
        alloc_s += time.perf_counter() - t0
        return LaunchResult(time.perf_counter() - t_start, compute_s, 0.0, alloc_s, reduced, trace)

    s = plan.shape
    lib = _lib.load()
    t0 = time.perf_counter()
    # SHARED (and check mode, which reads the arrays on the device) needs
    # device-addressable arrays: pinned sets as they are, others registered
    # for this launch only (ScatteredPatchSet.addressable: a lasting
    # registration of heap pages would break other buffers' pageable
    # copies).  COPY / POOLED over arrays that are not addressable run
    # host-staged: the library gathers chunks into pinned memory on the host
    # and DMAs them (fvb_launch_table) -- no registration.
    needs_map = transfer_mode is TransferMode.SHARED or ctx.check
    with (scattered.addressable(sync) if needs_map else contextlib.nullcontext()):
        alloc_s += time.perf_counter() - t0
        t0 = time.perf_counter()
        if ctx.check:
            _admissible(s, scattered.input_view(), ctx.params.gamma)
        handle, _ = _plan_handle(buffers.scratch, realization)
        shared = transfer_mode is TransferMode.SHARED
        red = ctypes.c_double()
        comp = ctypes.c_double()
        stream = torch.cuda.current_stream()
        _lib.check(lib.fvb_launch_table(
            FLAVOUR_OF[realization], LAYOUT_CODES[layout], s.dim, s.patch_size, s.patch_count,
            scattered.input_table().ctypes.data, scattered.output_table().ctypes.data,
            None if shared else buffers.batch.input.data_ptr(),
            None if shared else buffers.batch.output.data_ptr(), handle, ctx.dt, ctx.h,
            ctx.params.gamma, int(plan.with_reduction), None, int(chunk_patches), ctypes.byref(red),
            ctypes.byref(comp), stream.cuda_stream))
        launch_s = time.perf_counter() - t0
        if ctx.check and plan.with_reduction:
            _admissible(s, scattered.output_view(), ctx.params.gamma)
        t0 = time.perf_counter()
    alloc_s += time.perf_counter() - t0  # unregistering a transient registration
    if shared:
        compute_s, transfer_s = launch_s, 0.0
    else:
        compute_s = min(comp.value, launch_s)
        transfer_s = launch_s - compute_s
    reduced = max(0.0, red.value) if plan.with_reduction else None
    trace = trace_of(realization, plan, gpu_kernel_launches(realization, plan))
    t0 = time.perf_counter()
    release_buffers(buffers, arena)
    alloc_s += time.perf_counter() - t0
    total_s = time.perf_counter() - t_start
    return LaunchResult(total_s, compute_s, transfer_s, alloc_s, reduced, trace)


def default_context(gamma: float = 1.4, dt: float = 1e-3, h: float = 0.1,
                    check: bool = False) -> TimeStepContext:
    """The reference benchmark's run parameters (bench.py:150-153)."""
    return TimeStepContext(dt, h, EulerParameters(gamma), check)
