"""Randomised parity sweep: seeded draws over the whole configuration space
of the C ABI's step -- dimension, patch size, patch count, device layout,
realisation, reduction on/off, per-patch maxima, run parameters (dt, h,
gamma) and per-patch rescalings of the state that push whole patches, or
single cells, outside the fast paths' certified range (tiny / huge
densities and momenta, exact zeros) -- each against the CPU oracle
(oracle/fv_oracle.c, the run_sequential restatement), bytes and eigenvalue
bits.  The draws are fixed by the seed, so a failure names a reproducible
case; the NaN-aware byte compare treats every NaN as equal (payloads are
not part of the reference's contract).
"""

import os

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

REALIZATIONS = ("patch-wise", "batched", "task-graph")
LAYOUTS = ("soa", "aosoa", "aos")
N_CASES = int(os.environ.get("FVB_RANDOM_CASES", "300"))  # scale up for soak runs


@pytest.fixture(scope="module")
def fvb(cuda):
    import paper_2306_16731_b200 as pkg

    pkg.load_library()
    return pkg


def _draw(i):
    """Case i of the sweep: (d, p, t, layout, realization, reduce, lam_patch, dt, h, gamma, seed, scales)."""
    r = np.random.default_rng(20261017 + i)
    d = int(r.choice([2, 3], p=[0.6, 0.4]))
    p = int(r.choice([2, 3, 4, 5, 6, 7, 8, 11, 16, 17, 32])) if d == 2 else int(r.integers(2, 11))
    t = int(r.choice([1, 2, 3, int(r.integers(4, 40)), int(r.integers(40, 400))]))
    layout = LAYOUTS[int(r.integers(0, 3))]
    realization = REALIZATIONS[int(r.integers(0, 3))]
    reduce = bool(r.random() < 0.8)
    lam_patch = reduce and bool(r.random() < 0.5)
    gamma = float(r.choice([1.4, 5.0 / 3.0, float(r.uniform(1.05, 2.0))]))
    h = float(10.0 ** r.uniform(-3, 0))
    dt = float(h * 10.0 ** r.uniform(-4, -1))
    seed = int(r.integers(0, 1 << 30))
    # per-patch rescaling: (patch, kind) -- the Euler equations are invariant
    # under rho -> a rho, m -> a m, E -> a E (same velocities and sound speed),
    # so a whole patch can be moved to any magnitude; a single cell is zeroed
    # or given a tiny density
    scales = []
    for _ in range(int(r.integers(0, 4))):
        kind = str(r.choice(["tiny", "huge", "subnormal-cell", "zero-cell", "neg-zero-momentum"]))
        scales.append((int(r.integers(0, t)), kind, int(r.integers(0, (p + 2) ** d))))
    return d, p, t, layout, realization, reduce, lam_patch, dt, h, gamma, seed, scales


def _field(d, p, t, seed, scales, gamma):
    q = oracle.init_field_soa(d, p, t, seed, gamma=gamma)
    n, m = d + 2, (p + 2) ** d
    q = q.reshape(n, t, m).copy()
    with np.errstate(over="ignore"):  # a patch rescaled twice may overflow to inf: IEEE on both sides
        _rescale(q, scales)
    return np.ascontiguousarray(q.reshape(-1))


def _rescale(q, scales):
    for patch, kind, cell in scales:
        if kind == "tiny":
            q[:, patch, :] *= 2.0 ** -600
        elif kind == "huge":
            q[:, patch, :] *= 2.0 ** 600
        elif kind == "subnormal-cell":
            q[0, patch, cell] = 5e-324
        elif kind == "zero-cell":
            q[:, patch, cell] = 0.0
        else:
            q[1, patch, cell] = -0.0


def _same_bits_nan_aware(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb)) and a[~na].tobytes() == b[~nb].tobytes()


def _same_scalar(x, y):
    return np.float64(x).tobytes() == np.float64(y).tobytes() or (np.isnan(x) and np.isnan(y))


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_case_matches_oracle(fvb, i):
    import torch

    d, p, t, layout, realization, reduce, lam_patch, dt, h, gamma, seed, scales = case = _draw(i)
    q = _field(d, p, t, seed, scales, gamma)
    ref = oracle.step_c(d, p, t, q, dt=dt, h=h, gamma=gamma, with_reduction=reduce, lam_patch=lam_patch)
    shape = fvb.BatchShape(d, p, t)
    soa = fvb.DeviceFieldView(torch.from_numpy(q).cuda(), shape, True)
    inp = fvb.relayout(soa, fvb.Layout(layout))
    out = fvb.DeviceFieldView(torch.full((shape.output_size,), float("nan"), dtype=torch.float64, device="cuda"),
                              shape, False, fvb.Layout(layout))
    ctx = fvb.TimeStepContext(dt, h, fvb.EulerParameters(gamma))
    plan = fvb.build_plan(shape, reduce)
    lp = torch.full((t,), -1.0, dtype=torch.float64, device="cuda") if lam_patch else None
    lam = fvb.step_async(fvb.Realization(realization), plan, inp, out, ctx, lam_patch=lp)
    torch.cuda.synchronize()
    got = fvb.relayout(out, fvb.Layout.SOA).tensor.cpu().numpy()
    assert _same_bits_nan_aware(got, ref[0]), case
    if reduce:
        assert _same_scalar(float(lam.item()), ref[1]), case
    else:
        assert lam is None, case
    if lam_patch:
        assert _same_bits_nan_aware(lp.cpu().numpy(), ref[2]), case


N_LAUNCH = int(os.environ.get("FVB_RANDOM_LAUNCHES", "40"))


def _draw_launch(i):
    r = np.random.default_rng(777_000 + i)
    d = int(r.choice([2, 3]))
    p = int(r.choice([2, 3, 4, 5, 8, 16])) if d == 2 else int(r.choice([2, 3, 4, 6, 8]))
    t = int(r.choice([1, 5, int(r.integers(6, 300))]))
    return dict(d=d, p=p, t=t, layout=LAYOUTS[int(r.integers(0, 3))],
                realization=REALIZATIONS[int(r.integers(0, 3))], pinned=bool(r.random() < 0.5),
                reduce=bool(r.random() < 0.8), chunk=int(r.choice([0, 1, 7, int(r.integers(8, 200))])),
                h=float(10.0 ** r.uniform(-2, 0)), cfl=float(10.0 ** r.uniform(-3, -1)),
                seed=int(r.integers(0, 1 << 30)), gamma=float(r.choice([1.4, float(r.uniform(1.1, 1.9))])))


@pytest.mark.parametrize("i", range(N_LAUNCH))
def test_random_run_launch_matches_oracle(fvb, i):
    """run_launch -- the reference's entry point -- on random host patch sets
    (pinned blocks or independently allocated arrays), every transfer mode,
    random chunking of the COPY / POOLED pipeline: per-patch output bytes and
    the eigenvalue against the oracle; the host arrays end unregistered."""
    c = _draw_launch(i)
    d, p, t = c["d"], c["p"], c["t"]
    dt = c["cfl"] * c["h"]
    q = oracle.init_field_soa(d, p, t, c["seed"], gamma=c["gamma"])
    ref = oracle.step_c(d, p, t, q, dt=dt, h=c["h"], gamma=c["gamma"], with_reduction=c["reduce"])
    ref_aos = oracle.soa_to_aos_patches(ref[0], d, p, t, False)
    shape = fvb.BatchShape(d, p, t)
    base = fvb.init_field(shape, seed=c["seed"], gamma=c["gamma"], pinned=c["pinned"])
    plan = fvb.build_plan(shape, c["reduce"])
    ctx = fvb.TimeStepContext(dt, c["h"], fvb.EulerParameters(c["gamma"]))
    for mode in fvb.TransferMode:
        trial = base.clone()
        res = fvb.run_launch(plan, trial, fvb.Layout(c["layout"]), fvb.Realization(c["realization"]), mode,
                             fvb.ReductionStrategy.GROUP_TREE, ctx, fvb.DeviceArena(), chunk_patches=c["chunk"])
        assert np.concatenate(trial.outputs).tobytes() == ref_aos.tobytes(), (c, mode)
        if c["reduce"]:
            assert np.float64(res.reduced).tobytes() == np.float64(ref[1]).tobytes(), (c, mode)
        else:
            assert res.reduced is None, (c, mode)
        if not c["pinned"]:
            assert not trial.is_device_accessible(), (c, mode)
