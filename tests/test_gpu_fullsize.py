"""Whole-batch parity at BASELINE.json's full sizes.

Every byte of every output and every per-patch eigenvalue of the C2 / C3 /
C4 / C5-shard workloads against the CPU oracle (oracle/fv_oracle.c, the
literal run_sequential restatement pinned to the reference's own outputs by
tests/test_oracle.py), in every GPU realisation and with both eigenvalue
reductions: the filtered one (the fused kernels' default without per-patch
maxima) and the exhaustive one (FVB_TUNE_REDUCE_FILTER=0; and whenever
per-patch maxima are requested).  The oracle runs once per workload on the
host cores (OpenMP); its output is uploaded once and compared on the device.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

REALIZATIONS = ("patch-wise", "batched", "task-graph")


@pytest.fixture(scope="module")
def fvb(cuda):
    import paper_2306_16731_b200 as pkg

    pkg.load_library()
    return pkg


def _host_ram_bytes() -> int:
    try:
        import psutil

        return int(psutil.virtual_memory().available)
    except Exception:  # pragma: no cover
        return 0


def _reference(fvb, d, p, t, seed):
    """Device input (the reference's init_field bits) + the oracle's output,
    eigenvalue and per-patch maxima (output / maxima uploaded to the GPU)."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    q = fvb.init_field_device(shape, seed)
    q_host = q.tensor.cpu().numpy()
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q_host, lam_patch=True,
                                             threads=oracle.default_threads())
    del q_host
    ref_dev = torch.from_numpy(ref_out).cuda()
    del ref_out
    return shape, q, ref_dev, ref_red, torch.from_numpy(ref_lp).cuda()


def _check_all_modes(fvb, shape, q, ref_dev, ref_red, ref_lp, realizations):
    import torch

    ctx = fvb.default_context()
    plan = fvb.build_plan(shape, True)
    out = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False)
    lp = torch.empty(shape.patch_count, dtype=torch.float64, device="cuda")
    for real in realizations:
        r = fvb.Realization(real)
        for mode in ("filtered", "exhaustive", "per-patch"):
            out.tensor.fill_(float("nan"))
            lp.fill_(-1.0)
            if mode == "exhaustive":
                with fvb._lib.tuning(fvb._lib.FVB_TUNE_REDUCE_FILTER, 0):
                    lam = fvb.step_async(r, plan, q, out, ctx)
                    torch.cuda.synchronize()
            else:
                lam = fvb.step_async(r, plan, q, out, ctx, lam_patch=lp if mode == "per-patch" else None)
            torch.cuda.synchronize()
            where = f"{shape} {real} {mode}"
            assert torch.equal(out.tensor, ref_dev), where
            red = float(lam.item())
            assert red.hex() == ref_red.hex(), where
            if mode == "per-patch":
                assert torch.equal(lp, ref_lp), where
        fvb._lib.load().fvb_release_all()  # cascade / graph scratch


def test_c2_whole_batch(fvb):
    """C2: 2D p=3, 100k patches -- all flavours, both reductions."""
    shape, q, ref, red, lp = _reference(fvb, 2, 3, 100_000, 0)
    _check_all_modes(fvb, shape, q, ref, red, lp, REALIZATIONS)


@pytest.mark.parametrize("log2t", [10, 12, 14, 16, 18, 20])
def test_c3_sweep_whole_batch(fvb, log2t):
    """C3: 2D p=16, T = 2^10 .. 2^20 (the headline workload at the top)."""
    shape, q, ref, red, lp = _reference(fvb, 2, 16, 1 << log2t, 0)
    _check_all_modes(fvb, shape, q, ref, red, lp, REALIZATIONS)


def test_c4_whole_batch(fvb):
    """C4: 3D p=8, 100k patches -- all flavours, both reductions."""
    shape, q, ref, red, lp = _reference(fvb, 3, 8, 100_000, 0)
    _check_all_modes(fvb, shape, q, ref, red, lp, REALIZATIONS)


def test_3d_p6_whole_batch(fvb):
    """3D p=6, 100k patches (the 64-thread slot kernel, 28 stand-in
    threads) -- all flavours, both reductions."""
    shape, q, ref, red, lp = _reference(fvb, 3, 6, 100_000, 0)
    _check_all_modes(fvb, shape, q, ref, red, lp, REALIZATIONS)


def test_c5_2d_shard_whole_batch(fvb):
    """C5's per-GPU 2D shard: 4 Mi patches of 16x16 on one GPU (SoA offsets
    past 2^32), the fused flavour (the sharded bench's), both reductions.
    Needs ~80 GB of host RAM for the oracle's input and output."""
    import torch

    t = 4 << 20
    need = 8 * 4 * (18 * 18 + 16 * 16) * t + (8 << 30)
    if _host_ram_bytes() < need:
        pytest.skip(f"host RAM below {need / 2**30:.0f} GiB")
    shape, q, ref, red, lp = _reference(fvb, 2, 16, t, 0)
    assert 4 * t * 18 * 18 > 2**32
    _check_all_modes(fvb, shape, q, ref, red, lp, ("patch-wise",))
    del q, ref
    torch.cuda.empty_cache()
