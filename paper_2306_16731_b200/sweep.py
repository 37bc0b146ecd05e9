"""Benchmark sweeps in the reference's record / CSV schema (f3 row).

Mirror of pkg/src/patchbench/bench.py:136-206 and :323-414: ``BenchConfig``
(same fields and defaults, GPU realisations), ``BenchRecord`` with the
normalised ``time_per_volume_update_s`` / ``time_per_unknown_update_s``,
``run_sweep`` (configs in lexicographic order, one warm-up launch, then
``samples`` timed launches through ``run_launch``) and ``emit_csv`` with the
reference's 17-column header and 17-significant-digit floats.

``verify_against_golden`` is the device form of the reference's
``verify_against_sequential`` (bench.py:262-320): the golden run is the
literal per-step realisation -- the cascade kernels (one per reference
step, IEEE double) with the hook-free physics policy (EulerPlain: no fast
paths, no reduce filter), AoS, SHARED, check=True -- and the trial must
match it byte for byte, or ``VerifyError`` names the first differing patch
and offset.  (The CPU oracle that pins both to the reference lives in the
test suite; the product never imports it.)
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _lib
from .context import TimeStepContext
from .equations import EulerParameters
from .errors import VerifyError
from .executors import GpuScratch, Realization, ReductionStrategy
from .kernelgraph import build_plan
from .launch import init_field, run_launch
from .memory import DeviceArena, ScatteredPatchSet, TransferMode
from .patchdata import BatchShape, Layout

__all__ = ["CSV_HEADER", "BenchConfig", "BenchRecord", "run_sweep", "emit_csv", "verify_against_golden"]

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


def _first_mismatch(golden: ScatteredPatchSet, got: ScatteredPatchSet) -> str | None:
    """bench.py:262-268: the first differing output value."""
    for patch, (a, b) in enumerate(zip(golden.outputs, got.outputs)):
        a, b = np.asarray(a), np.asarray(b)
        if a.tobytes() != b.tobytes():
            bad = np.nonzero(~(a == b))[0]
            idx = int(bad[0]) if bad.size else 0
            return f"patch {patch} offset {idx}: golden {a[idx]!r}, got {b[idx]!r}"
    return None


def verify_against_golden(plan, scattered: ScatteredPatchSet, config: BenchConfig,
                          arena: DeviceArena, pool=None) -> None:
    """Run the configuration once and demand bitwise equality with the
    golden run (module docstring); raises VerifyError with the first
    mismatch (bench.py:271-320)."""
    params = EulerParameters(config.gamma)
    golden = scattered.clone()
    with _lib.physics(_lib.FVB_PHYSICS_EULER_PLAIN), _lib.tuning(_lib.FVB_TUNE_REDUCE_FILTER, 0):
        golden_reduced = run_launch(plan, golden, Layout.AOS, Realization.BATCHED, TransferMode.SHARED,
                                    config.reduction_strategy, TimeStepContext(config.dt, config.h, params, True),
                                    DeviceArena(), pool, config.workgroup_limit).reduced
    trial = scattered.clone()
    result = run_launch(plan, trial, config.layout, config.realization, config.transfer_mode,
                        config.reduction_strategy, TimeStepContext(config.dt, config.h, params, False),
                        arena, pool, config.workgroup_limit)
    mismatch = _first_mismatch(golden, trial)
    if mismatch is not None:
        raise VerifyError(f"{config}: output differs from the golden run at {mismatch}")
    if plan.with_reduction:
        if np.float64(golden_reduced).tobytes() != np.float64(result.reduced).tobytes():
            raise VerifyError(f"{config}: reduced eigenvalue {result.reduced!r} != golden "
                              f"{golden_reduced!r}")


def run_sweep(configs: Iterable[BenchConfig], verify: bool = False,
              log: Callable[[str], None] | None = None) -> list[BenchRecord]:
    """Time every configuration; records in lexicographic configuration order.
    verify=True first checks each configuration against the golden run
    (verify_against_golden, raising VerifyError)."""
    records = []
    ordered = sorted(configs, key=lambda c: c.sort_key)
    for i, cfg in enumerate(ordered):
        shape = cfg.shape
        plan = build_plan(shape, cfg.with_reduction)
        patches = init_field(shape, cfg.seed, cfg.gamma)
        arena = DeviceArena()
        ctx = TimeStepContext(cfg.dt, cfg.h, EulerParameters(cfg.gamma))

        if verify:
            verify_against_golden(plan, patches, cfg, arena)

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
