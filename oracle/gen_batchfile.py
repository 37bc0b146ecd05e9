"""Batch-file fixtures written by the REFERENCE's dump_batch (this container only).

    python oracle/gen_batchfile.py

Imports patchbench read-only from /root/reference/pkg/src: init_field
(bench.py:107-133) -> run_launch(SEQUENTIAL, SHARED) for the golden outputs
-> gather the inputs (memory.gather_patches) and the outputs (the inverse of
memory.scatter_results, same offset tables) into a PatchBatch in the given
layout -> patchdata.dump_batch (patchdata.py:337-351).  The files pin
paper_2306_16731_b200.memory.read_batch_file / write_batch_file / load_batch /
dump_batch to the reference's on-disk format (tests/test_host.py,
tests/test_gpu_api.py).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
CASES = [("2d_p3_t5_soa", 2, 3, 5, 7, "soa"), ("3d_p2_t3_aosoa", 3, 2, 3, 8, "aosoa"),
         ("2d_p4_t2_aos", 2, 4, 2, 9, "aos")]


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    from patchbench.bench import init_field, run_launch
    from patchbench.equations import EulerParameters
    from patchbench.executors import Realization, ReductionStrategy, WorkerPool
    from patchbench.kernelgraph import build_plan
    from patchbench.memory import DeviceArena, TransferMode, gather_patches
    from patchbench.microkernels import TimeStepContext
    from patchbench.patchdata import (BatchShape, FlatFieldView, Layout, PatchBatch, dump_batch,
                                      offset_table)

    for name, d, p, t, seed, lay in CASES:
        shape = BatchShape(d, p, t)
        layout = Layout(lay)
        sc = init_field(shape, seed, 1.4)
        with WorkerPool(1) as pool:
            run_launch(build_plan(shape, True), sc, Layout.AOS, Realization.SEQUENTIAL, TransferMode.SHARED,
                       ReductionStrategy.GROUP_TREE, TimeStepContext(1e-3, 0.1, EulerParameters(1.4), True),
                       DeviceArena(), pool)
        batch = PatchBatch(shape, layout, np.zeros(shape.input_size), np.zeros(shape.output_size))
        gather_patches(sc, batch)
        one = BatchShape(d, p, 1)
        src_offs = offset_table(Layout.AOS, one, haloed=False).ravel()
        dst_table = offset_table(layout, shape, haloed=False).ravel()
        view = FlatFieldView(batch.output, layout, shape, haloed=False)
        for patch, arr in enumerate(sc.outputs):
            _, base = view.block(patch)
            batch.output[base + dst_table] = arr[src_offs]
        path = OUT / f"batch_{name}.bin"
        dump_batch(batch, path)
        print(path, path.stat().st_size)


if __name__ == "__main__":
    main()
