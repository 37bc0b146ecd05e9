"""Generate golden fixtures by running the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Imports the reference package ``patchbench`` read-only from
/root/reference/pkg/src, runs its golden executor ``run_sequential``
(pkg/src/patchbench/executors.py:219-270; ``run_batched`` for the larger
cases, byte-identical per pkg/tests/test_acceptance.py:67-114) through its
own entry point ``run_launch`` (pkg/src/patchbench/bench.py:209-259) in
SHARED mode on AoS scattered patches, and writes

* tests/golden/golden.json -- one record per case: shape, seed, run
  parameters, reduced eigenvalue (repr + IEEE hex), SHA-256 of the
  concatenated per-patch AoS input and output arrays;
* tests/golden/small_cases.npz -- raw AoS input/output arrays of the small
  cases, so tests can diff element-wise without regenerating inputs.

/root/reference never exists on the GPU box; these committed fixtures are
what travels.  Rerunning this script must reproduce them byte for byte.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT_DIR = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    from patchbench.bench import init_field, run_launch
    from patchbench.equations import EulerParameters
    from patchbench.executors import Realization, ReductionStrategy, WorkerPool
    from patchbench.kernelgraph import build_plan
    from patchbench.memory import DeviceArena, TransferMode, allocate_scattered
    from patchbench.microkernels import TimeStepContext
    from patchbench.patchdata import BatchShape, Layout

    def constant(shape, q):
        sc = allocate_scattered(shape)
        for arr in sc.inputs:
            arr[:] = np.tile(np.asarray(q, dtype=np.float64), shape.haloed_cells)
        return sc

    cases = []
    # acceptance matrix seeds (pkg/tests/test_acceptance.py:72-78)
    for d in (2, 3):
        for p in (4, 6, 8):
            for t in (1, 4, 16):
                cases.append(dict(d=d, p=p, t=t, seed=d * 100 + p * 10))
    # BASELINE configs, full or scaled down
    cases += [
        dict(d=2, p=16, t=64, seed=0, tag="C1"),
        dict(d=2, p=3, t=1000, seed=0, tag="C2-subset", realization="batched"),
        dict(d=2, p=16, t=1024, seed=0, tag="C3-point", realization="batched"),
        dict(d=3, p=8, t=64, seed=0, tag="C4-subset", realization="batched"),
    ]
    # edge cases: smallest patch, odd p, non-default run parameters, no reduction
    cases += [
        dict(d=2, p=2, t=3, seed=7, tag="p2"),
        dict(d=3, p=2, t=2, seed=8, tag="p2-3d"),
        dict(d=2, p=3, t=5, seed=9, tag="p3"),
        dict(d=2, p=5, t=3, seed=10, tag="p5"),
        dict(d=3, p=3, t=2, seed=11, tag="p3-3d"),
        dict(d=2, p=4, t=2, seed=12, gamma=5.0 / 3.0, dt=2.5e-3, h=0.05, tag="params"),
        dict(d=3, p=4, t=2, seed=13, gamma=1.3, dt=7e-4, h=0.2, tag="params-3d"),
        dict(d=2, p=6, t=3, seed=14, with_reduction=False, tag="noreduce"),
        dict(d=3, p=4, t=2, seed=15, with_reduction=False, tag="noreduce-3d"),
        dict(d=2, p=32, t=2, seed=16, tag="p32"),
        dict(d=2, p=17, t=2, seed=17, tag="p17"),
        dict(d=2, p=4, t=2, const=(1.3, 0.26, -0.39, 3.25), tag="constant"),
        dict(d=3, p=4, t=2, const=(1.3, 0.26, -0.39, 0.13, 3.25), tag="constant-3d"),
    ]

    records = []
    arrays = {}
    with WorkerPool(4) as pool:
        for c in cases:
            d, p, t = c["d"], c["p"], c["t"]
            gamma = c.get("gamma", 1.4)
            dt = c.get("dt", 1e-3)
            h = c.get("h", 0.1)
            with_reduction = c.get("with_reduction", True)
            shape = BatchShape(d, p, t)
            if "const" in c:
                scattered = constant(shape, c["const"])
            else:
                scattered = init_field(shape, c["seed"], gamma)
            realization = (Realization.BATCHED if c.get("realization") == "batched"
                           else Realization.SEQUENTIAL)
            ctx = TimeStepContext(dt, h, EulerParameters(gamma), check=True)
            t0 = time.perf_counter()
            result = run_launch(build_plan(shape, with_reduction), scattered, Layout.AOS,
                                realization, TransferMode.SHARED,
                                ReductionStrategy.GROUP_TREE, ctx, DeviceArena(), pool)
            elapsed = time.perf_counter() - t0
            inp = np.concatenate(scattered.inputs)
            out = np.concatenate(scattered.outputs)
            name = c.get("tag", f"d{d}p{p}t{t}s{c.get('seed')}")
            rec = dict(
                name=name, d=d, p=p, t=t, seed=c.get("seed"), const=c.get("const"),
                gamma=gamma, dt=dt, h=h, with_reduction=with_reduction,
                realization=realization.value,
                reduced=None if result.reduced is None else repr(result.reduced),
                reduced_hex=None if result.reduced is None else float(result.reduced).hex(),
                sha256_in=hashlib.sha256(inp.astype("<f8").tobytes()).hexdigest(),
                sha256_out=hashlib.sha256(out.astype("<f8").tobytes()).hexdigest(),
            )
            records.append(rec)
            if out.size <= 4096:
                arrays[name + "/in"] = inp
                arrays[name + "/out"] = out
            print(f"{name}: reduced={rec['reduced']} in={rec['sha256_in'][:16]} "
                  f"out={rec['sha256_out'][:16]} ({elapsed:.2f}s)")
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    (OUT_DIR / "golden.json").write_text(json.dumps(records, indent=1) + "\n")
    np.savez_compressed(OUT_DIR / "small_cases.npz", **arrays)


if __name__ == "__main__":
    main()
