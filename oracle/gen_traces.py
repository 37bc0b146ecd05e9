"""Trace / arena-counter fixtures from the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_traces.py

Runs the reference's parallel realisations through its own ``run_launch``
(pkg/src/patchbench/bench.py:209-259) over the acceptance matrix shapes
(pkg/tests/test_acceptance.py:72-78) and records, per (d, p, T,
realisation, with_reduction), the ExecutionTrace integers the reference
returns (executors.py:79-87, filled at :344-347, :438-445, :528-534), and
the DeviceArena allocation counters per transfer mode after 1 and 3 launches
(memory.py:105-137, pkg/tests/test_acceptance.py:220-258).  Writes
tests/golden/traces.json; the GPU tests compare the repo's run_launch with
it field for field.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "traces.json"


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    from patchbench.bench import init_field, run_launch
    from patchbench.equations import EulerParameters
    from patchbench.executors import Realization, ReductionStrategy, WorkerPool
    from patchbench.kernelgraph import build_plan
    from patchbench.memory import DeviceArena, TransferMode
    from patchbench.microkernels import TimeStepContext
    from patchbench.patchdata import BatchShape, Layout

    ctx = TimeStepContext(1e-3, 0.1, EulerParameters(1.4))
    traces = []
    counters = []
    with WorkerPool(2) as pool:
        for d in (2, 3):
            for p in (4, 6, 8):
                for t in (1, 4, 16):
                    shape = BatchShape(d, p, t)
                    base = init_field(shape, seed=d * 100 + p * 10)
                    for realization in (Realization.PATCH_WISE, Realization.BATCHED,
                                        Realization.TASK_GRAPH):
                        for with_reduction in (True, False):
                            tr = run_launch(build_plan(shape, with_reduction), base.clone(), Layout.AOS,
                                            realization, TransferMode.SHARED,
                                            ReductionStrategy.GROUP_TREE, ctx, DeviceArena(),
                                            pool).trace
                            traces.append(dict(
                                d=d, p=p, t=t, realization=realization.value,
                                with_reduction=with_reduction,
                                global_sync_count=tr.global_sync_count,
                                per_step_task_counts=list(tr.per_step_task_counts),
                                masked_invocation_count=tr.masked_invocation_count,
                                executed_invocation_count=tr.executed_invocation_count,
                                launch_count=tr.launch_count))
        for d, p, t in ((2, 4, 2), (3, 4, 2)):
            shape = BatchShape(d, p, t)
            base = init_field(shape, seed=4)
            for mode in TransferMode:
                for layout in Layout:
                    arena = DeviceArena()
                    counts = []
                    for _ in range(3):
                        run_launch(build_plan(shape, True), base.clone(), layout,
                                   Realization.BATCHED, mode, ReductionStrategy.GROUP_TREE, ctx,
                                   arena, pool)
                        counts.append(arena.allocation_count)
                    counters.append(dict(d=d, p=p, t=t, mode=mode.value, layout=layout.value,
                                         allocation_counts=counts,
                                         outstanding_zero=arena.outstanding_bytes == 0
                                         if mode is TransferMode.EXPLICIT_COPY else None))
    OUT.write_text(json.dumps(dict(traces=traces, arena_counters=counters), indent=1) + "\n")
    print(f"{len(traces)} traces, {len(counters)} counter records -> {OUT}")


if __name__ == "__main__":
    main()
