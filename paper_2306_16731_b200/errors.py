"""Exception classes with the reference's names and bases, so callers that
catch the reference's errors keep working (pkg/src/patchbench/equations.py:38-39,
executors.py:74-76, kernelgraph.py:43-44, memory.py:56-57, bench.py:85-86)."""


class InvalidStateError(ValueError):
    """A conserved state violates admissibility (rho <= 0 or p <= 0)."""


class WorkgroupLimitError(RuntimeError):
    """The patch does not fit one fused work unit (the reference's emulated
    workgroup limit, or the B200 kernel's shared-memory budget)."""


class GraphCycleError(RuntimeError):
    """The task DAG contains a cycle (never happens for built plans)."""


class ShapeMismatchError(ValueError):
    """Scattered set and batch disagree on their shape."""


class VerifyError(RuntimeError):
    """A GPU realisation's output differs from the golden CPU run."""
