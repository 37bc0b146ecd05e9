"""Batch layouts (§8 f4): AoS / SoA / AoSoA device batches (patchdata.py:49-58,
142-168) run natively by every flavour, bit-identical to the oracle.

Inputs are the reference's seeded fields; the oracle computes in SoA and the
device results are permuted back to SoA (fvb_relayout) before comparing bytes.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

REALIZATIONS = ("patch-wise", "batched", "task-graph")
CASES = [(2, 16, 64, 0), (2, 3, 1000, 0), (2, 5, 37, 250), (2, 17, 9, 270), (2, 32, 5, 20),
         (3, 8, 16, 380), (3, 4, 33, 340), (3, 5, 7, 350), (3, 6, 11, 360)]


@pytest.fixture(scope="module")
def fvb(cuda):
    import paper_2306_16731_b200 as pkg

    pkg.load_library()
    return pkg


def _views(fvb, d, p, t, q_np, layout):
    import torch

    shape = fvb.BatchShape(d, p, t)
    soa = fvb.DeviceFieldView(torch.from_numpy(q_np).cuda(), shape, True)
    inp = fvb.relayout(soa, layout)
    out = fvb.DeviceFieldView(torch.full((shape.output_size,), float("nan"), dtype=torch.float64,
                                         device="cuda"), shape, False, layout)
    return shape, inp, out


@pytest.mark.parametrize("layout", ["aos", "aosoa", "soa"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "d%dp%dT%d" % c[:3])
@pytest.mark.parametrize("realization", REALIZATIONS)
def test_layout_bit_exact(fvb, layout, case, realization):
    import torch

    d, p, t, seed = case
    q = oracle.init_field_soa(d, p, t, seed)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    shape, inp, out = _views(fvb, d, p, t, q, fvb.Layout(layout))
    ctx = fvb.default_context()
    plan = fvb.build_plan(shape, True)
    real = fvb.Realization(realization)
    for lam_patch in (None, torch.empty(t, dtype=torch.float64, device="cuda")):
        lam = fvb.step_async(real, plan, inp, out, ctx, lam_patch=lam_patch)
        got = fvb.relayout(out, fvb.Layout.SOA).tensor.cpu().numpy()
        assert got.tobytes() == ref_out.tobytes()
        assert float(lam.item()) == ref_red
        if lam_patch is not None:
            assert lam_patch.cpu().numpy().tobytes() == ref_lp.tobytes()


@pytest.mark.parametrize("d,p,t", [(2, 4, 3), (3, 3, 2), (2, 16, 5)])
def test_relayout_matches_layout_enumerator(fvb, d, p, t):
    """fvb_relayout against the reference's linear_offset (patchdata.py:142-168)."""
    import itertools

    import torch

    for haloed in (True, False):
        shape = fvb.BatchShape(d, p, t)
        n = shape.input_size if haloed else shape.output_size
        src = torch.arange(n, dtype=torch.float64, device="cuda")
        soa = fvb.DeviceFieldView(src, shape, haloed)
        m = shape.extent(haloed)
        lo = -1 if haloed else 0
        cells = list(itertools.product(range(lo, lo + m), repeat=d))
        for lay in fvb.Layout:
            got = fvb.relayout(soa, lay).tensor.cpu().numpy()
            back = fvb.relayout(fvb.relayout(soa, lay), fvb.Layout.SOA).tensor
            assert torch.equal(back, src)
            for patch in (0, t - 1):
                for cell in cells[:: max(1, len(cells) // 17)]:
                    for k in range(d + 2):
                        c = tuple(reversed(cell))  # product() varies the last coordinate fastest
                        s = fvb.linear_offset(fvb.Layout.SOA, shape, haloed, patch, c, k)
                        o = fvb.linear_offset(lay, shape, haloed, patch, c, k)
                        assert got[o] == float(s)


@pytest.mark.parametrize("layout", ["aos", "aosoa"])
def test_run_launch_layouts(fvb, layout):
    """run_launch gathers into the requested device layout (AoS: straight DMA)."""
    shape = fvb.BatchShape(3, 4, 9)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    q = oracle.init_field_soa(3, 4, 9, 340)
    ref_out, ref_red = oracle.step_c(3, 4, 9, q)
    arena = fvb.DeviceArena()
    for mode in (fvb.TransferMode.EXPLICIT_COPY, fvb.TransferMode.POOLED):
        for real in fvb.Realization.PATCH_WISE, fvb.Realization.BATCHED, fvb.Realization.TASK_GRAPH:
            sc = fvb.init_field(shape, 340)
            res = fvb.run_launch(plan, sc, fvb.Layout(layout), real, mode,
                                 fvb.ReductionStrategy.GROUP_TREE, ctx, arena)
            assert res.reduced == ref_red
            assert np.concatenate(sc.outputs).tobytes() == \
                oracle.soa_to_aos_patches(ref_out, 3, 4, 9, False).tobytes()


def test_mixed_layouts_rejected(fvb):
    import torch

    shape = fvb.BatchShape(2, 4, 2)
    inp = fvb.DeviceFieldView(torch.zeros(shape.input_size, dtype=torch.float64, device="cuda"),
                              shape, True, fvb.Layout.AOS)
    out = fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False, fvb.Layout.SOA)
    with pytest.raises(ValueError):
        fvb.step_async(fvb.Realization.PATCH_WISE, fvb.build_plan(shape, True), inp, out,
                       fvb.default_context())


@pytest.mark.parametrize("variant", [0, 9])
@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (2, 5, 40), (2, 3, 21), (2, 7, 9)])
def test_aos_2d_copy_widths(fvb, variant, d, p, t):
    """2D AoS batches: unknown pairs by 16-byte cp.async (the default when
    aligned) and by 8-byte copies (FVB_TUNE_PENCIL_VARIANT = 9, also the
    path of per-patch pointer tables), bit-identical to the oracle."""
    import torch

    q = oracle.init_field_soa(d, p, t, 77 + p)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    shape, inp, out = _views(fvb, d, p, t, q, fvb.Layout.AOS)
    plan = fvb.build_plan(shape, True)
    lp = torch.empty(t, dtype=torch.float64, device="cuda")
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_PENCIL_VARIANT, variant):
        for lam_patch in (None, lp):
            lam = fvb.step_async(fvb.Realization.PATCH_WISE, plan, inp, out, fvb.default_context(), lam_patch=lam_patch)
            got = fvb.relayout(out, fvb.Layout.SOA).tensor.cpu().numpy()
            assert got.tobytes() == ref_out.tobytes()
            assert float(lam.item()) == ref_red
    assert lp.cpu().numpy().tobytes() == ref_lp.tobytes()
