"""Small launches of every kernel family, checked against the CPU oracle.

Run under compute-sanitizer (scripts/sanitize.sh): racecheck / memcheck /
synccheck see each kernel once on a batch small enough for the tools.
Each case prints one line "CASE <name>: ok" (or raises).

    python scripts/sanitize_cases.py [--only SUBSTRING]
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16731_b200 as fvb  # noqa: E402
from oracle import oracle  # noqa: E402  (checker only)


def step(real, d, p, t, layout=fvb.Layout.SOA, lam_patch=False, seed=3, offset=0):
    shape = fvb.BatchShape(d, p, t)
    q = oracle.init_field_soa(d, p, t, seed)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    base = torch.empty(shape.input_size + offset, dtype=torch.float64, device="cuda")
    qd = base[offset:]
    qd.copy_(torch.from_numpy(q))
    inp = fvb.DeviceFieldView(qd, shape, True)
    if layout is not fvb.Layout.SOA:
        inp = fvb.relayout(inp, layout)
    out = fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False, layout)
    plan = fvb.build_plan(shape, True)
    lp = torch.zeros(t, dtype=torch.float64, device="cuda") if lam_patch else None
    lam = fvb.step_async(fvb.Realization(real), plan, inp, out, fvb.default_context(),
                         lam_patch=lp)
    torch.cuda.synchronize()
    if layout is not fvb.Layout.SOA:
        out = fvb.relayout(out, fvb.Layout.SOA)
    got = out.tensor.cpu().numpy()
    assert got.tobytes() == ref_out.tobytes(), f"{real} d={d} p={p} t={t} {layout}: output"
    assert float(lam.item()) == ref_red, f"{real} d={d} p={p} t={t}: eigenvalue"
    if lam_patch:
        assert lp.cpu().numpy().tobytes() == ref_lp.tobytes()


def plain(fn):
    """Run fn with the hook-free physics policy (EulerPlain)."""
    def run():
        with fvb._lib.physics(fvb._lib.FVB_PHYSICS_EULER_PLAIN):
            fn()
        fvb._lib.load().fvb_release_all()
    return run


def launch(real, d, p, t, mode, layout="soa", chunk=0, seed=4, pinned=False):
    shape = fvb.BatchShape(d, p, t)
    q = oracle.init_field_soa(d, p, t, seed)
    ref_out, ref_red = oracle.step_c(d, p, t, q)
    sc = fvb.init_field(shape, seed, pinned=pinned)
    res = fvb.run_launch(fvb.build_plan(shape, True), sc, fvb.Layout(layout), fvb.Realization(real),
                         fvb.TransferMode(mode), fvb.ReductionStrategy.GROUP_TREE,
                         fvb.default_context(), fvb.DeviceArena(), chunk_patches=chunk)
    got = np.concatenate(sc.outputs)
    assert got.tobytes() == oracle.soa_to_aos_patches(ref_out, d, p, t, False).tobytes(), (real, mode)
    assert res.reduced == ref_red


def slab5(fn):
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_SLAB_VARIANT, 5):
        fn()


CASES = {
    "fused2d_tma_p16": lambda: step("patch-wise", 2, 16, 40),
    "fused2d_tma_p8_aosoa": lambda: step("patch-wise", 2, 8, 20, fvb.Layout.AOSOA),
    "fused2d_tile_p3": lambda: step("patch-wise", 2, 3, 50),
    "fused2d_tile_p3_lampatch": lambda: step("patch-wise", 2, 3, 66, lam_patch=True),
    "fused2d_cpasync_p3_odd": lambda: step("patch-wise", 2, 3, 51),
    "fused2d_cpasync_p5_lampatch": lambda: step("patch-wise", 2, 5, 13, lam_patch=True),
    "fused2d_cpasync_p16_aos": lambda: step("patch-wise", 2, 16, 10, fvb.Layout.AOS),
    "fused2d_cpasync_p16_unaligned": lambda: step("patch-wise", 2, 16, 9, offset=1),
    "fused3d_warp_p8": lambda: step("patch-wise", 3, 8, 6),
    "fused3d_warp_p8_lampatch": lambda: step("patch-wise", 3, 8, 5, lam_patch=True),
    "fused3d_warp_p8_aos": lambda: step("patch-wise", 3, 8, 3, fvb.Layout.AOS),  # AoS plane map
    "fused3d_slab_p8_variant5": lambda: slab5(lambda: step("patch-wise", 3, 8, 3)),  # two-warp slot kernel
    "fused3d_slab_p6_aos": lambda: step("patch-wise", 3, 6, 3, fvb.Layout.AOS),
    "fused3d_slab_p4": lambda: step("patch-wise", 3, 4, 7),  # sub-warp slots: 2 patches per warp
    "fused3d_slab_p3_lampatch": lambda: step("patch-wise", 3, 3, 9, lam_patch=True),
    "fused3d_slab_p2": lambda: step("patch-wise", 3, 2, 11),  # 4 patches per warp
    "fused3d_slab_p5": lambda: step("patch-wise", 3, 5, 5),
    "fused_generic_2d_p20": lambda: step("patch-wise", 2, 20, 3),
    "fused_generic_2d_p40": lambda: step("patch-wise", 2, 40, 2),
    "cascade_2d_p6": lambda: step("batched", 2, 6, 9, lam_patch=True),
    "cascade_3d_p4": lambda: step("batched", 3, 4, 4),
    "graph_2d_p4": lambda: step("task-graph", 2, 4, 5),
    "graph_3d_p4": lambda: step("task-graph", 3, 4, 3),
    # run_launch over per-patch host arrays: SHARED (pointer-table step
    # kernels on registered memory) and the chunked COPY pipeline (table
    # gather / scatter kernels)
    "launch_shared_2d_p16": lambda: launch("patch-wise", 2, 16, 9, "shared"),
    "launch_shared_3d_p8": lambda: launch("patch-wise", 3, 8, 3, "shared"),
    "launch_shared_cascade_3d_p4": lambda: launch("batched", 3, 4, 3, "shared"),
    "launch_shared_graph_2d_p4": lambda: launch("task-graph", 2, 4, 3, "shared"),
    "launch_copy_2d_p16_soa": lambda: launch("patch-wise", 2, 16, 9, "copy", chunk=4),  # host-staged
    "launch_staged_graph_3d_p4_aos": lambda: launch("task-graph", 3, 4, 7, "pooled", "aos", chunk=2),
    "launch_pooled_3d_p8_aosoa": lambda: launch("batched", 3, 8, 3, "pooled", "aosoa", chunk=2),
    # pinned blocks: chunk DMA + device permutation (fvb_launch_table)
    "launch_dma_2d_p16_soa": lambda: launch("patch-wise", 2, 16, 9, "pooled", chunk=4, pinned=True),
    "launch_dma_graph_3d_p4_aos": lambda: launch("task-graph", 3, 4, 5, "copy", "aos", chunk=2, pinned=True),
    # the hook-free physics policy through the fused kernels
    "plain_fused2d_tma_p16": plain(lambda: step("patch-wise", 2, 16, 40)),
    "plain_fused2d_tile_p3": plain(lambda: step("patch-wise", 2, 3, 34)),
    "plain_fused3d_warp_p8": plain(lambda: step("patch-wise", 3, 8, 4)),
}


def main() -> None:
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else ""
    fvb.load_library()
    for name, fn in CASES.items():
        if only and only not in name:
            continue
        fn()
        print(f"CASE {name}: ok", flush=True)


if __name__ == "__main__":
    main()
