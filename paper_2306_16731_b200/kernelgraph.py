"""Algorithmic steps, per-step ranges and the per-patch task DAG.

Host mirror of pkg/src/patchbench/kernelgraph.py: the step order
(copy, flux_0..d-1, lambda_0..d-1, acc_0..d-1, [reduce], :173-182), the
per-step range sizes (:134-149), the per-patch DAG (:215-247) and its Kahn
check (:257-271).  On the GPU the step structure is compiled into the
kernels; this plan object carries the shape for the drop-in signatures, the
trace counters and the task-graph flavour's node structure (the CUDA graph
built in csrc/fvb.cu follows exactly these edges, lifted to patch chunks).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .errors import GraphCycleError
from .patchdata import BatchShape

__all__ = ["StepOp", "StepKind", "StepSpec", "TaskDag", "KernelPlan", "step_sequence",
           "range_size", "build_task_graph", "build_plan", "topological_order",
           "invocations_per_patch", "masked_per_patch"]


class StepOp(Enum):
    COPY = "copy"
    FLUX = "flux"
    EIGENVALUE = "lambda"
    ACCUMULATE = "acc"
    REDUCE = "reduce"


_DIRECTIONAL = (StepOp.FLUX, StepOp.EIGENVALUE, StepOp.ACCUMULATE)


@dataclass(frozen=True)
class StepKind:
    op: StepOp
    axis: int | None = None

    def __post_init__(self) -> None:
        if (self.op in _DIRECTIONAL) != (self.axis is not None):
            raise ValueError(f"{self.op.value} step axis mismatch: {self.axis}")

    @property
    def name(self) -> str:
        return self.op.value if self.axis is None else f"{self.op.value}_{'xyz'[self.axis]}"


def range_size(shape: BatchShape, kind: StepKind) -> int:
    """Cells per patch of a step: p^d, or (p+2)p^(d-1) for flux/lambda."""
    p, d = shape.patch_size, shape.dim
    if kind.op in (StepOp.FLUX, StepOp.EIGENVALUE):
        return (p + 2) * p ** (d - 1)
    return p**d


@dataclass(frozen=True)
class StepSpec:
    kind: StepKind
    range_size: int


@dataclass
class TaskDag:
    """(patch, step) nodes; edges never cross patches."""

    shape: BatchShape
    with_reduction: bool
    steps: list[StepKind]
    edges: list[tuple[int, int]]
    successors: list[list[int]]
    indegree: list[int]

    @property
    def node_count(self) -> int:
        return self.shape.patch_count * len(self.steps)

    def node_id(self, patch: int, step_index: int) -> int:
        return patch * len(self.steps) + step_index


@dataclass
class KernelPlan:
    shape: BatchShape
    with_reduction: bool
    steps: list[StepSpec]
    dag: TaskDag | None = field(default=None, repr=False)


def step_sequence(shape: BatchShape, with_reduction: bool) -> list[StepKind]:
    axes = range(shape.dim)
    seq = [StepKind(StepOp.COPY)]
    for op in (StepOp.FLUX, StepOp.EIGENVALUE, StepOp.ACCUMULATE):
        seq.extend(StepKind(op, a) for a in axes)
    if with_reduction:
        seq.append(StepKind(StepOp.REDUCE))
    return seq


def per_patch_edges(shape: BatchShape, with_reduction: bool) -> list[tuple[int, int]]:
    """Edges of one patch's DAG as (src step index, dst step index)."""
    seq = step_sequence(shape, with_reduction)
    at = {k: i for i, k in enumerate(seq)}
    copy = at[StepKind(StepOp.COPY)]
    edges = []
    for a in range(shape.dim):
        acc = at[StepKind(StepOp.ACCUMULATE, a)]
        edges += [(copy, acc), (at[StepKind(StepOp.FLUX, a)], acc),
                  (at[StepKind(StepOp.EIGENVALUE, a)], acc)]
        if a:
            edges.append((at[StepKind(StepOp.ACCUMULATE, a - 1)], acc))
    if with_reduction:
        edges.append((at[StepKind(StepOp.ACCUMULATE, shape.dim - 1)], at[StepKind(StepOp.REDUCE)]))
    return edges


def build_task_graph(shape: BatchShape, with_reduction: bool) -> TaskDag:
    seq = step_sequence(shape, with_reduction)
    local = per_patch_edges(shape, with_reduction)
    n = len(seq)
    total = shape.patch_count * n
    succ: list[list[int]] = [[] for _ in range(total)]
    indeg = [0] * total
    edges = []
    for patch in range(shape.patch_count):
        for s, t in local:
            u, v = patch * n + s, patch * n + t
            edges.append((u, v))
            succ[u].append(v)
            indeg[v] += 1
    return TaskDag(shape, with_reduction, seq, edges, succ, indeg)


def build_plan(shape: BatchShape, with_reduction: bool, with_dag: bool = False) -> KernelPlan:
    """Step specs in serialized order (+ the full per-patch DAG on request;
    it is T*(1+3d+1) nodes, so it is only materialised when asked for)."""
    steps = [StepSpec(k, range_size(shape, k)) for k in step_sequence(shape, with_reduction)]
    dag = build_task_graph(shape, with_reduction) if with_dag else None
    return KernelPlan(shape, with_reduction, steps, dag)


def topological_order(dag: TaskDag) -> list[int]:
    indeg = list(dag.indegree)
    ready = [v for v, k in enumerate(indeg) if k == 0]
    order = []
    while ready:
        v = ready.pop()
        order.append(v)
        for w in dag.successors[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                ready.append(w)
    if len(order) != dag.node_count:
        raise GraphCycleError(f"cycle among {dag.node_count - len(order)} nodes")
    return order


def invocations_per_patch(shape: BatchShape, with_reduction: bool) -> int:
    return sum(range_size(shape, k) for k in step_sequence(shape, with_reduction))


def masked_per_patch(shape: BatchShape, with_reduction: bool) -> int:
    """Union-range lanes an emulated (p+2)^d workgroup would mask per patch."""
    return sum(shape.haloed_cells - range_size(shape, k)
               for k in step_sequence(shape, with_reduction))
