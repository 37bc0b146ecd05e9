"""Benchmark sweeps in the reference's record / CSV schema (f3 row).

Mirror of pkg/src/patchbench/bench.py:136-206 and :323-414: ``BenchConfig``
(same fields and defaults, GPU realisations), ``BenchRecord`` with the
normalised ``time_per_volume_update_s`` / ``time_per_unknown_update_s``,
``run_sweep`` (configs in lexicographic order, one warm-up launch, then
``samples`` timed launches through ``run_launch``) and ``emit_csv`` with the
reference's 17-column header and 17-significant-digit floats.  The golden
cross-check of the reference's ``verify_against_sequential`` lives in the
test suite (it needs the CPU oracle, which the product never imports).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

from .context import TimeStepContext
from .equations import EulerParameters
from .executors import GpuScratch, Realization, ReductionStrategy
from .kernelgraph import build_plan
from .launch import init_field, run_launch
from .memory import DeviceArena, TransferMode
from .patchdata import BatchShape, Layout

__all__ = ["CSV_HEADER", "BenchConfig", "BenchRecord", "run_sweep", "emit_csv"]

CSV_HEADER = [
    "dim", "p", "T", "layout", "realization", "transfer_mode", "reduction_strategy",
    "with_reduction", "samples", "workers", "mean_total_s", "mean_compute_s",
    "mean_transfer_s", "mean_alloc_s", "time_per_volume_update_s",
    "time_per_unknown_update_s", "reduced_eigenvalue",
]


@dataclass(frozen=True)
class BenchConfig:
    dim: int = 2
    patch_size: int = 4
    patch_count: int = 4
    layout: Layout = Layout.SOA
    realization: Realization = Realization.PATCH_WISE
    transfer_mode: TransferMode = TransferMode.POOLED
    reduction_strategy: ReductionStrategy = ReductionStrategy.GROUP_TREE
    with_reduction: bool = True
    samples: int = 16
    workers: int = 1  # the GPU is the pool; kept for the schema
    gamma: float = 1.4
    dt: float = 1e-3
    h: float = 1e-1
    seed: int = 0
    workgroup_limit: int = 1024

    @property
    def shape(self) -> BatchShape:
        return BatchShape(self.dim, self.patch_size, self.patch_count)

    @property
    def sort_key(self) -> tuple:
        return (self.dim, self.patch_size, self.patch_count, self.layout.value,
                self.realization.value, self.transfer_mode.value, self.reduction_strategy.value,
                self.with_reduction, self.samples, self.workers)


@dataclass
class BenchRecord:
    config: BenchConfig
    mean_total_s: float
    mean_compute_s: float
    mean_transfer_s: float
    mean_alloc_s: float
    min_total_s: float
    reduced_eigenvalue: float

    @property
    def time_per_volume_update_s(self) -> float:
        s = self.config.shape
        return self.mean_total_s / (s.patch_count * s.interior_cells)

    @property
    def time_per_unknown_update_s(self) -> float:
        s = self.config.shape
        return self.mean_total_s / (s.patch_count * s.interior_cells * s.unknowns)


def run_sweep(configs: Iterable[BenchConfig],
              log: Callable[[str], None] | None = None) -> list[BenchRecord]:
    """Time every configuration; records in lexicographic configuration order."""
    records = []
    ordered = sorted(configs, key=lambda c: c.sort_key)
    for i, cfg in enumerate(ordered):
        shape = cfg.shape
        plan = build_plan(shape, cfg.with_reduction)
        patches = init_field(shape, cfg.seed, cfg.gamma)
        arena = DeviceArena()
        ctx = TimeStepContext(cfg.dt, cfg.h, EulerParameters(cfg.gamma))

        def launch():
            return run_launch(plan, patches, cfg.layout, cfg.realization, cfg.transfer_mode,
                              cfg.reduction_strategy, ctx, arena, None, cfg.workgroup_limit)

        launch()  # warm-up; primes the pooled arena and instantiates graphs
        results = [launch() for _ in range(cfg.samples)]
        n = len(results)
        reduced = results[-1].reduced
        rec = BenchRecord(cfg, sum(r.total_s for r in results) / n,
                          sum(r.compute_s for r in results) / n,
                          sum(r.transfer_s for r in results) / n,
                          sum(r.alloc_s for r in results) / n,
                          min(r.total_s for r in results),
                          0.0 if reduced is None else reduced)
        records.append(rec)
        if log is not None:
            log(f"[{i + 1}/{len(ordered)}] d={cfg.dim} p={cfg.patch_size} T={cfg.patch_count} "
                f"{cfg.realization.value} {cfg.transfer_mode.value} "
                f"mean_total={rec.mean_total_s:.3e}s")
    return records


def _fmt(x: float) -> str:
    return f"{x:.17g}"


def emit_csv(records: Sequence[BenchRecord], path: str, extended: bool = False) -> None:
    header = list(CSV_HEADER) + (["min_total_s"] if extended else [])
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(header)
        for r in records:
            c = r.config
            row = [c.dim, c.patch_size, c.patch_count, c.layout.value, c.realization.value,
                   c.transfer_mode.value, c.reduction_strategy.value,
                   "true" if c.with_reduction else "false", c.samples, c.workers,
                   _fmt(r.mean_total_s), _fmt(r.mean_compute_s), _fmt(r.mean_transfer_s),
                   _fmt(r.mean_alloc_s), _fmt(r.time_per_volume_update_s),
                   _fmt(r.time_per_unknown_update_s), _fmt(r.reduced_eigenvalue)]
            if extended:
                row.append(_fmt(r.min_total_s))
            w.writerow(row)
