"""B200-native batched multi-patch finite-volume step (arXiv 2306.16731).

Rusanov finite volumes for the compressible Euler equations over batches of
Cartesian patches with one-cell halos, computed by hand-written sm_100a CUDA
kernels (libfvb.so, C ABI in include/fvb.h) behind the reference package's
Python API (``patchbench``): ``run_launch``, the executor signatures
``run_batched`` / ``run_patchwise`` / ``run_taskgraph`` and the user
microkernel interface ``flux`` / ``max_eigenvalue``.

There is no CPU fallback: importing the compute path loads libfvb.so and
fails loudly when it is missing.  The CPU oracle used by the tests lives in
``oracle/`` and is never imported from here.
"""

from . import _lib
from .context import TimeStepContext
from .equations import EulerParameters, flux, is_admissible, max_eigenvalue, pressure
from .errors import (GraphCycleError, InvalidStateError, ShapeMismatchError, VerifyError,
                     WorkgroupLimitError)
from .executors import (ExecutionTrace, GpuScratch, Realization, ReductionStrategy, reduce_max,
                        run_batched, run_patchwise, run_taskgraph, step_async)
from .kernelgraph import KernelPlan, build_plan, build_task_graph, step_sequence
from .launch import (LaunchResult, admissible_dt, default_context, init_field, init_field_device,
                     run_launch)
from .memory import (DeviceArena, DeviceBatch, DevicePatchSet, GpuScratchArrays, HostPatchView,
                     ScatteredPatchSet, TransferMode, allocate_scattered, dump_batch, gather_patches,
                     load_batch, scatter_results)
from .patchdata import LAYOUT_CODES, BatchShape, DeviceFieldView, Layout, linear_offset, relayout

__version__ = "0.1.0"

__all__ = [
    "BatchShape", "DeviceArena", "DeviceBatch", "GpuScratchArrays", "HostPatchView",
    "gather_patches", "scatter_results", "dump_batch", "load_batch", "DeviceFieldView", "DevicePatchSet", "EulerParameters",
    "ExecutionTrace", "GpuScratch", "GraphCycleError", "InvalidStateError", "KernelPlan",
    "LAYOUT_CODES", "Layout", "LaunchResult", "linear_offset", "relayout", "Realization", "ReductionStrategy", "ScatteredPatchSet",
    "ShapeMismatchError", "TimeStepContext", "TransferMode", "VerifyError",
    "WorkgroupLimitError", "admissible_dt", "allocate_scattered", "build_plan",
    "build_task_graph", "default_context", "flux", "init_field", "init_field_device",
    "is_admissible", "max_eigenvalue", "pressure", "reduce_max", "run_batched", "run_launch",
    "run_patchwise", "run_taskgraph", "step_async", "step_sequence", "load_library",
]


def load_library():
    """Load libfvb.so (raises if it is missing -- no fallback)."""
    return _lib.load()
