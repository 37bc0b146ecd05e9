"""GPU realisations of the batched FV step behind the reference's executor API.

Drop-in signatures of pkg/src/patchbench/executors.py:

* ``run_patchwise(plan, inp, out, scratch, ctx, pool, strategy, workgroup_limit)``
  (:390-445) -> the fused nested-parallel kernel (FVB_FUSED);
* ``run_batched(plan, inp, out, scratch, ctx, pool, strategy)`` (:312-382) ->
  the per-step kernel cascade (FVB_CASCADE);
* ``run_taskgraph(plan, inp, out, scratch, ctx, pool, strategy, prebuilt_dag)``
  (:453-535) -> a CUDA Graph over the per-step kernels following the lifted
  per-patch DAG (FVB_GRAPH).

``inp`` / ``out`` are :class:`DeviceFieldView` s (SoA float64 CUDA tensors);
each call returns ``(reduced | None, ExecutionTrace)`` like the reference,
where ``reduced`` is the max eigenvalue of the updated solution as a Python
float (the only host synchronisation).  ``pool`` is accepted and ignored (the
GPU is the pool).  All ``ReductionStrategy`` values give the identical bits:
max is exact, and the kernels always reduce warp-shuffle -> CTA -> one 64-bit
atomicMax per warp.  ``step_async`` is the stream-ordered form that leaves the
eigenvalue on the device (used by the benchmark and the multi-GPU driver).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

from . import _lib
from .context import TimeStepContext
from .errors import InvalidStateError, WorkgroupLimitError
from .kernelgraph import KernelPlan, StepOp, masked_per_patch  # noqa: F401  (re-export)
from .patchdata import LAYOUT_CODES, BatchShape, DeviceFieldView, Layout, relayout

__all__ = ["Realization", "ReductionStrategy", "ExecutionTrace", "WorkgroupLimitError",
           "GpuScratch", "run_batched", "run_patchwise", "run_taskgraph", "step_async",
           "reduce_max", "trace_of", "NEUTRAL_EIGENVALUE", "FLAVOUR_OF"]

NEUTRAL_EIGENVALUE = 0.0


class Realization(Enum):
    SEQUENTIAL = "sequential"  # the CPU golden run; lives in oracle/, not here
    PATCH_WISE = "patch-wise"
    BATCHED = "batched"
    TASK_GRAPH = "task-graph"


class ReductionStrategy(Enum):
    GROUP_TREE = "tree"
    SHARED_MAX = "shared-max"
    SERIAL = "serial"


FLAVOUR_OF = {
    Realization.PATCH_WISE: _lib.FVB_FUSED,
    Realization.BATCHED: _lib.FVB_CASCADE,
    Realization.TASK_GRAPH: _lib.FVB_GRAPH,
}


@dataclass
class ExecutionTrace:
    """Scheduling telemetry of one launch (executors.py:79-87) with the
    reference's integers (trace_of); gpu_kernel_launches is the GPU's own
    count of enqueued kernels."""

    global_sync_count: int = 0
    per_step_task_counts: list[int] = field(default_factory=list)
    masked_invocation_count: int = 0
    executed_invocation_count: int = 0
    launch_count: int = 0
    gpu_kernel_launches: int = 0  # CUDA kernels / graph kernel nodes actually enqueued


class GpuScratch:
    """Library-owned scratch arena + graph of one (flavour, shape).

    The GPU analogue of ScratchArrays (microkernels.py:70-112): cascade and
    graph flavours keep per-axis flux / wave-speed temporaries in HBM, sized
    tight to the flux range; the fused flavour needs none.  ``chunks`` splits
    the task graph into that many independent per-chunk step chains.
    """

    def __init__(self, shape: BatchShape, realization: Realization, chunks: int = 1) -> None:
        if realization not in FLAVOUR_OF:
            raise ValueError(f"{realization} is not a GPU realisation")
        lib = _lib.load()
        self.shape = shape
        self.realization = realization
        self.flavour = FLAVOUR_OF[realization]
        handle = ctypes.c_void_p()
        _lib.check(lib.fvb_plan_create(self.flavour, shape.dim, shape.patch_size,
                                       shape.patch_count, int(chunks), ctypes.byref(handle)))
        self.handle = handle

    def graph_nodes(self) -> int:
        n = ctypes.c_int64()
        _lib.check(_lib.load().fvb_plan_graph_nodes(self.handle, ctypes.byref(n)))
        return n.value

    def kernel_launches(self, with_reduction: bool) -> int:
        n = ctypes.c_int64()
        _lib.check(_lib.load().fvb_plan_kernel_launches(self.handle, int(with_reduction),
                                                        ctypes.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.load().fvb_plan_destroy(self.handle)
            self.handle = None

    def __del__(self) -> None:  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def _check_views(plan: KernelPlan, inp, out) -> None:
    from .memory import HostPatchView

    if isinstance(inp, HostPatchView) or isinstance(out, HostPatchView):
        if not (isinstance(inp, HostPatchView) and isinstance(out, HostPatchView)):
            raise TypeError("host patch views (SHARED mode) come in pairs")
        if inp.patches is not out.patches or inp.shape != plan.shape or not inp.haloed or out.haloed:
            raise ValueError("host patch views do not match the plan's shape / extents")
        return
    if not isinstance(inp, DeviceFieldView) or not isinstance(out, DeviceFieldView):
        raise TypeError("GPU realisations take DeviceFieldView (or SHARED HostPatchView) operands")
    if inp.shape != plan.shape or out.shape != plan.shape or not inp.haloed or out.haloed:
        raise ValueError("field views do not match the plan's shape / extents")
    if inp.layout is not out.layout:
        raise ValueError(f"input is {inp.layout.value}, output {out.layout.value}: one batch layout")
    a, b = inp.tensor, out.tensor
    if a.device != b.device:
        raise ValueError(f"input on {a.device}, output on {b.device}: one device")
    a0, b0 = a.data_ptr(), b.data_ptr()
    if a0 < b0 + b.numel() * b.element_size() and b0 < a0 + a.numel() * a.element_size():
        raise ValueError("input and output batches overlap (a step never writes its input)")


def _admissible(shape: BatchShape, view, gamma: float) -> None:
    """check=True mode (equations.py:64-73): raise on rho <= 0 or p <= 0 in
    the states the reference's step evaluates -- the flux ranges of the
    input (no corner halo cells) or the interior output (reduce)."""
    import torch

    from .memory import HostPatchView

    if isinstance(view, HostPatchView):
        dev = torch.device("cuda", torch.cuda.current_device())
        tab = view.device_table(dev)
        q_ptr, tab_ptr, layout = None, tab.data_ptr(), Layout.AOS
    else:
        dev = view.tensor.device
        tab = None
        q_ptr, tab_ptr, layout = view.data_ptr(), None, view.layout
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.load().fvb_check_admissible_ex(shape.dim, shape.patch_size, shape.patch_count,
                                                   int(view.haloed), LAYOUT_CODES[layout], gamma, q_ptr,
                                                   tab_ptr, bad.data_ptr(), stream))
    n = int(bad.item())
    if n:
        what = "input" if view.haloed else "updated"
        raise InvalidStateError(f"{n} {what} cells with non-positive density or pressure")


def _plan_handle(scratch, realization: Realization):
    """The libfvb plan a launch runs on: a GpuScratch's own, an arena's
    GpuScratchArrays bound to a plan, or None (library cache / stateless)."""
    from .memory import GpuScratchArrays

    if isinstance(scratch, GpuScratch):
        if scratch.flavour != FLAVOUR_OF[realization]:
            raise ValueError("scratch was created for another realisation")
        return scratch.handle, scratch.shape
    if isinstance(scratch, GpuScratchArrays) and realization is not Realization.PATCH_WISE:
        return scratch.plan(FLAVOUR_OF[realization]).handle, scratch.shape
    return None, None


def step_async(realization: Realization, plan: KernelPlan, inp, out, ctx: TimeStepContext,
               scratch=None, lam=None, lam_patch=None, stream=None, dt_dev=None, dt_patch=None):
    """Enqueue one step on ``stream`` (default: torch's current stream).

    Returns the device tensor holding the reduced eigenvalue (``lam``, one
    float64, allocated if None) or None without reduction.  No host sync.
    ``inp`` / ``out``: DeviceFieldViews of a batch in HBM, or HostPatchViews
    of a ScatteredPatchSet (SHARED mode: computed in place on the per-patch
    arrays through pointer tables).  ``scratch``: None, a GpuScratch, or an
    arena's GpuScratchArrays.  ``dt_dev``: a one-element float64 CUDA
    tensor holding dt (then ``ctx.dt`` is ignored and the kernels form dt/h
    on the device, fvb_step_dt) -- the form a CUDA-graph-captured
    multi-step loop uses.  ``dt_patch``: a T-element float64 CUDA tensor of
    per-patch time steps (local time stepping, fvb_step_lts).
    """
    import torch

    from .memory import HostPatchView

    _check_views(plan, inp, out)
    if realization not in FLAVOUR_OF:
        raise ValueError(f"{realization} has no GPU flavour (the sequential run is the CPU oracle)")
    lib = _lib.load()
    s = plan.shape
    tables = isinstance(inp, HostPatchView)
    dev = torch.device("cuda", torch.cuda.current_device()) if tables else inp.tensor.device
    with torch.cuda.device(dev):  # the library launches on the current device
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        if plan.with_reduction and lam is None:
            lam = torch.empty(1, dtype=torch.float64, device=dev)
        if lam is not None and plan.with_reduction:
            if lam.dtype != torch.float64 or not lam.is_cuda or lam.numel() < 1 or lam.device != dev:
                raise ValueError("lam must be a float64 CUDA tensor on the batch's device")
        if lam_patch is not None and plan.with_reduction:
            if (lam_patch.dtype != torch.float64 or not lam_patch.is_cuda or lam_patch.device != dev
                    or lam_patch.numel() < s.patch_count or not lam_patch.is_contiguous()):
                raise ValueError("lam_patch must be a contiguous float64 CUDA tensor with one entry per patch")
        lam_ptr = lam.data_ptr() if plan.with_reduction else None
        lp_ptr = lam_patch.data_ptr() if (plan.with_reduction and lam_patch is not None) else None
        flavour = FLAVOUR_OF[realization]
        layout = LAYOUT_CODES[Layout.AOS if tables else inp.layout]
        handle, sshape = _plan_handle(scratch, realization)
        if handle is not None and sshape != s:
            raise ValueError("scratch was created for another shape")
        in_tab = out_tab = None
        if tables:
            in_tab, out_tab = inp.device_table(dev), out.device_table(dev)
        if dt_patch is not None or dt_dev is not None:
            if handle is not None or tables:
                raise ValueError("dt_dev / dt_patch run on device batches with the library's cached plans")
            if dt_patch is not None:
                if dt_dev is not None:
                    raise ValueError("pass dt_dev or dt_patch, not both")
                if dt_patch.numel() != s.patch_count or dt_patch.dtype != torch.float64 or not dt_patch.is_cuda:
                    raise ValueError("dt_patch must be a float64 CUDA tensor with one dt per patch")
                _lib.check(lib.fvb_step_lts(flavour, layout, s.dim, s.patch_size, s.patch_count,
                                            inp.data_ptr(), out.data_ptr(), dt_patch.data_ptr(), ctx.h,
                                            ctx.params.gamma, int(plan.with_reduction), lam_ptr, lp_ptr,
                                            stream.cuda_stream))
            else:
                _lib.check(lib.fvb_step_dt(flavour, layout, s.dim, s.patch_size, s.patch_count,
                                           inp.data_ptr(), out.data_ptr(), dt_dev.data_ptr(), ctx.h,
                                           ctx.params.gamma, int(plan.with_reduction), lam_ptr, lp_ptr,
                                           stream.cuda_stream))
            return lam if plan.with_reduction else None
        run = (ctx.dt, ctx.h, ctx.params.gamma, int(plan.with_reduction), lam_ptr, lp_ptr,
               stream.cuda_stream)
        if handle is not None:
            _lib.check(lib.fvb_plan_set_layout(handle, layout))
            _lib.check(lib.fvb_plan_execute_ex(handle, None if tables else inp.data_ptr(),
                                               None if tables else out.data_ptr(),
                                               in_tab.data_ptr() if tables else None,
                                               out_tab.data_ptr() if tables else None, 0, -1, 1, *run))
        elif tables:
            _lib.check(lib.fvb_step_table(flavour, s.dim, s.patch_size, s.patch_count, in_tab.data_ptr(),
                                          out_tab.data_ptr(), *run))
        else:
            _lib.check(lib.fvb_step_layout(flavour, layout, s.dim, s.patch_size, s.patch_count,
                                           inp.data_ptr(), out.data_ptr(), *run))
        return lam if plan.with_reduction else None


def _run(realization, plan, inp, out, scratch, ctx):
    import contextlib

    import torch

    from .memory import HostPatchView

    held = contextlib.ExitStack()
    with held:
        if isinstance(inp, HostPatchView):  # SHARED: the sets addressable for this run only
            for view in (inp, out):
                held.enter_context(view.patches.addressable(torch.cuda.synchronize))
        if ctx.check:
            _admissible(plan.shape, inp, ctx.params.gamma)
        lam = step_async(realization, plan, inp, out, ctx, scratch)
        if ctx.check and plan.with_reduction:  # the reduce evaluates the updated states
            _admissible(plan.shape, out, ctx.params.gamma)
        return None if lam is None else float(lam.item())


def trace_of(realization: Realization, plan: KernelPlan, kernel_launches: int = 0) -> ExecutionTrace:
    """The reference's ExecutionTrace integers for a realisation
    (executors.py:344-347, :438-445, :528-534): batched = one global sync and
    launch per step; patch-wise = one sync, one launch, T*masked_per_patch
    masked lanes of the union-range region; task graph = one sync and one
    launch per DAG node (T*steps).  ``kernel_launches`` adds what the GPU
    actually enqueued (CUDA kernels or graph kernel nodes)."""
    t = plan.shape.patch_count
    per_step = [t * s.range_size for s in plan.steps]
    n = len(plan.steps)
    if realization is Realization.BATCHED:
        syncs, masked, launches = n, 0, n
    elif realization is Realization.PATCH_WISE:
        syncs, masked, launches = 1, t * masked_per_patch(plan.shape, plan.with_reduction), 1
    elif realization is Realization.TASK_GRAPH:
        syncs, masked, launches = 1, 0, t * n
    else:
        raise ValueError(f"{realization} has no GPU trace")
    return ExecutionTrace(global_sync_count=syncs, per_step_task_counts=per_step,
                          masked_invocation_count=masked, executed_invocation_count=sum(per_step),
                          launch_count=launches, gpu_kernel_launches=kernel_launches)


def gpu_kernel_launches(realization: Realization, plan: KernelPlan) -> int:
    """Kernels one GPU launch enqueues: fused 1, cascade one per step, graph
    one kernel node per step (per chunk of a chunked GpuScratch graph)."""
    n = len(plan.steps)
    return {Realization.PATCH_WISE: 1, Realization.BATCHED: n, Realization.TASK_GRAPH: n}[realization]


def run_patchwise(plan, inp, out, scratch, ctx, pool=None,
                  strategy: ReductionStrategy = ReductionStrategy.GROUP_TREE,
                  workgroup_limit: int = 1024):
    """Fused nested-parallel kernel: all steps of a patch in one launch."""
    union = plan.shape.haloed_cells
    if union > workgroup_limit:
        raise WorkgroupLimitError(
            f"(p+2)^d = {union} exceeds workgroup limit {workgroup_limit}; "
            "the patch must be broken down manually")
    reduced = _run(Realization.PATCH_WISE, plan, inp, out, scratch, ctx)
    return reduced, trace_of(Realization.PATCH_WISE, plan, 1)


def run_batched(plan, inp, out, scratch, ctx, pool=None,
                strategy: ReductionStrategy = ReductionStrategy.GROUP_TREE):
    """One kernel per step, stream-ordered (a device-wide wait after each)."""
    reduced = _run(Realization.BATCHED, plan, inp, out, scratch, ctx)
    return reduced, trace_of(Realization.BATCHED, plan, len(plan.steps))


def run_taskgraph(plan, inp, out, scratch, ctx, pool=None,
                  strategy: ReductionStrategy = ReductionStrategy.GROUP_TREE,
                  prebuilt_dag: bool = False):
    """CUDA Graph over the per-step kernels along the lifted per-patch DAG.

    With a GpuScratch / arena scratch the graph is instantiated once per
    scratch and replayed; without one the library caches it per (shape,
    stream).  The trace counts the DAG's T*steps nodes like the reference.
    """
    reduced = _run(Realization.TASK_GRAPH, plan, inp, out, scratch, ctx)
    if isinstance(scratch, GpuScratch):
        launches = scratch.kernel_launches(plan.with_reduction)
    else:
        launches = len(plan.steps)
    return reduced, trace_of(Realization.TASK_GRAPH, plan, launches)


def reduce_max(values, strategy: ReductionStrategy = ReductionStrategy.GROUP_TREE,
               pool=None) -> float:
    """max(0, max(values)) -- exact for every strategy (executors.py:162-183)."""
    import torch

    v = torch.as_tensor(values, dtype=torch.float64)
    if v.numel() == 0:
        return NEUTRAL_EIGENVALUE
    return max(NEUTRAL_EIGENVALUE, float(v.max().item()))
