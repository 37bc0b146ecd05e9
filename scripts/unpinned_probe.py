"""run_launch on independently allocated (unpinned) host arrays: time split
per transfer mode (registration is per launch, see memory.py)."""
import time

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2306_16731_b200 as fvb

for t in (1 << 12, 1 << 16):
    shape = fvb.BatchShape(2, 16, t)
    sc = fvb.init_field(shape, 0, pinned=False)
    plan = fvb.build_plan(shape, True)
    arena = fvb.DeviceArena()
    for mode in fvb.TransferMode:
        fvb.run_launch(plan, sc, fvb.Layout.SOA, fvb.Realization.PATCH_WISE, mode,
                       fvb.ReductionStrategy.GROUP_TREE, fvb.default_context(), arena)
        t0 = time.perf_counter()
        r = fvb.run_launch(plan, sc, fvb.Layout.SOA, fvb.Realization.PATCH_WISE, mode,
                           fvb.ReductionStrategy.GROUP_TREE, fvb.default_context(), arena)
        el = time.perf_counter() - t0
        gb = t * 8 * 4 * (324 + 256) / 1e9
        print(f"T={t:6d} {mode.value:7s} total {r.total_s*1e3:8.2f} ms (alloc/register {r.alloc_s*1e3:7.2f}, "
              f"transfer {r.transfer_s*1e3:7.2f}, compute {r.compute_s*1e3:6.2f}) {gb / el:6.1f} GB/s of host data",
              flush=True)
