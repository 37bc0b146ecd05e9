"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north star): eigenvalue bit-exact; Q_new within 1e-12 relative -- and
in practice bit-exact, which is what these tests demand (assert on bytes),
since the kernels keep the reference's expression trees and --fmad=false.
Inputs are the reference's seeded fields, generated on the device by the
jump-ahead LCG and checked against the oracle's generator bit for bit.
"""

import hashlib

import numpy as np
import pytest

from golden_cases import case_input_soa, records
from oracle import oracle

pytestmark = pytest.mark.gpu

REALIZATIONS = ("patch-wise", "batched", "task-graph")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def fvb(cuda):
    import paper_2306_16731_b200 as pkg

    pkg.load_library()
    return pkg


def _step(fvb, realization, d, p, t, q_np=None, q_dev=None, dt=1e-3, h=0.1, gamma=1.4,
          with_reduction=True, scratch=None, lam_patch=False):
    import torch

    shape = fvb.BatchShape(d, p, t)
    if q_dev is None:
        q_dev = torch.from_numpy(np.ascontiguousarray(q_np)).cuda()
    inp = fvb.DeviceFieldView(q_dev, shape, True)
    out = fvb.DeviceFieldView(torch.full((shape.output_size,), float("nan"), dtype=torch.float64,
                                         device="cuda"), shape, False)
    ctx = fvb.TimeStepContext(dt, h, fvb.EulerParameters(gamma))
    plan = fvb.build_plan(shape, with_reduction)
    real = fvb.Realization(realization)
    lp = torch.full((t,), -1.0, dtype=torch.float64, device="cuda") if lam_patch else None
    lam = fvb.step_async(real, plan, inp, out, ctx, scratch=scratch, lam_patch=lp)
    torch.cuda.synchronize()
    red = None if lam is None else float(lam.item())
    res = (out.tensor.cpu().numpy(), red)
    return res + ((lp.cpu().numpy(),) if lam_patch else ())


@pytest.mark.parametrize("rec", records(), ids=lambda r: r["name"])
@pytest.mark.parametrize("realization", REALIZATIONS)
def test_golden_cases_bit_exact(fvb, rec, realization):
    d, p, t = rec["d"], rec["p"], rec["t"]
    q = case_input_soa(rec, oracle)
    out, red = _step(fvb, realization, d, p, t, q, dt=rec["dt"], h=rec["h"], gamma=rec["gamma"],
                     with_reduction=rec["with_reduction"])
    assert _sha(oracle.soa_to_aos_patches(out, d, p, t, False)) == rec["sha256_out"]
    if rec["with_reduction"]:
        assert red.hex() == rec["reduced_hex"]
    else:
        assert red is None


@pytest.mark.parametrize("d,p,t,seed", [(2, 16, 64, 0), (2, 3, 1000, 0), (3, 8, 64, 0),
                                        (2, 7, 33, 5), (2, 31, 5, 6), (2, 40, 3, 7),
                                        (3, 5, 9, 8), (3, 10, 2, 9), (2, 2, 129, 10)])
@pytest.mark.parametrize("realization", REALIZATIONS)
def test_matches_oracle_with_per_patch_eigenvalues(fvb, d, p, t, seed, realization):
    q = oracle.init_field_soa(d, p, t, seed)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    out, red, lp = _step(fvb, realization, d, p, t, q, lam_patch=True)
    assert out.tobytes() == ref_out.tobytes()
    assert red == ref_red and red.hex() == ref_red.hex()
    assert lp.tobytes() == ref_lp.tobytes()


@pytest.mark.parametrize("d,p,t,seed", [(2, 16, 1000, 3), (3, 8, 100, 4), (2, 3, 5000, 5),
                                        (3, 2, 77, 6)])
def test_device_field_generator_matches_init_field(fvb, d, p, t, seed):
    import torch

    shape = fvb.BatchShape(d, p, t)
    q = fvb.init_field_device(shape, seed)
    torch.cuda.synchronize()
    assert q.tensor.cpu().numpy().tobytes() == oracle.init_field_soa(d, p, t, seed).tobytes()
    # a shard of the same stream
    part = fvb.init_field_device(fvb.BatchShape(d, p, t - t // 3), seed, patch_begin=t // 3)
    whole = q.as_array()[:, t // 3:, :].contiguous().view(-1)
    assert torch.equal(part.tensor, whole)


def test_microkernel_probe_matches_host_equations(fvb):
    import torch

    params = fvb.EulerParameters(1.4)
    rng = np.random.default_rng(0)
    lib = fvb.load_library()
    for d in (2, 3):
        n = d + 2
        count = 257
        prim = rng.uniform([0.5] + [-0.5] * d + [0.5], [2.0] + [0.5] * d + [2.0], (count, n))
        q = prim.copy()
        q[:, 1:d + 1] = prim[:, :1] * prim[:, 1:d + 1]
        q[:, -1] = prim[:, -1] / 0.4 + 0.5 * prim[:, 0] * (prim[:, 1:d + 1] ** 2).sum(1)
        q[:3] = 0.0  # zero states exercise the IEEE redo of the fast policy
        q[3, 1:d + 1] = -0.0
        q[4, 0] = 1e-300
        qd = torch.from_numpy(q.reshape(-1)).cuda()
        for axis in range(d):
            for policy in (0, 1):
                f = torch.empty(count * n, dtype=torch.float64, device="cuda")
                lam = torch.empty(count, dtype=torch.float64, device="cuda")
                assert lib.fvb_eval_microkernels(d, count, axis, 1.4, policy, qd.data_ptr(),
                                                 f.data_ptr(), lam.data_ptr(), None) == 0
                torch.cuda.synchronize()
                fh, lh = f.cpu().numpy().reshape(count, n), lam.cpu().numpy()
                for i in range(count):
                    with np.errstate(all="ignore"):
                        try:
                            ref_f = fvb.flux(tuple(q[i]), axis, params)
                            ref_l = fvb.max_eigenvalue(tuple(q[i]), axis, params)
                        except (ZeroDivisionError, ValueError):
                            continue  # Python raises where IEEE gives inf/nan
                    assert np.array(ref_f).tobytes() == fh[i].tobytes(), (i, policy)
                    assert np.float64(ref_l).tobytes() == lh[i].tobytes(), (i, policy)


def test_fast_math_policy_matches_ieee(fvb):
    """realx.cuh: where the XReal fast paths do not raise their flag, a/b and
    sqrt(a) equal IEEE bit for bit; the flag fires on the out-of-range cases."""
    import torch

    lib = fvb.load_library()
    rng = np.random.default_rng(7)
    n = 1 << 22
    a = np.concatenate([
        rng.uniform(-4, 4, n // 4),
        np.exp(rng.uniform(-700, 700, n // 4)) * rng.choice([-1, 1], n // 4),
        rng.standard_normal(n // 4) * 10.0 ** rng.integers(-320, 300, n // 4),
        np.frombuffer(rng.bytes(8 * (n // 4)), dtype=np.float64),  # random bit patterns
    ])
    b = np.concatenate([
        rng.uniform(0.5, 2.0, n // 4),
        np.exp(rng.uniform(-700, 700, n // 4)),
        rng.standard_normal(n // 4) * 10.0 ** rng.integers(-320, 300, n // 4),
        np.frombuffer(rng.bytes(8 * (n // 4)), dtype=np.float64),
    ])
    special = np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                        np.inf, -np.inf, np.nan, 1.0, -1.0, 3.0])
    sa, sb = np.meshgrid(special, special)
    a = np.concatenate([a, sa.ravel()])
    b = np.concatenate([b, sb.ravel()])
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    qd, rd = torch.empty_like(ad), torch.empty_like(ad)
    fl = torch.empty(a.size, dtype=torch.int32, device="cuda")
    assert lib.fvb_probe_fastmath(a.size, ad.data_ptr(), bd.data_ptr(), qd.data_ptr(),
                                  rd.data_ptr(), fl.data_ptr(), None) == 0
    torch.cuda.synchronize()
    with np.errstate(all="ignore"):
        ieee_r = np.sqrt(a)
    q, r, f = qd.cpu().numpy(), rd.cpu().numpy(), fl.cpu().numpy()
    okq, okr = (f & 1) == 0, (f & 2) == 0
    with np.errstate(all="ignore"):
        host_q = a / b
    assert np.array_equal(q[okq].view(np.int64), host_q[okq].view(np.int64))
    assert np.array_equal(r[okr].view(np.int64), ieee_r[okr].view(np.int64))
    assert okq[: n // 4].mean() > 0.999 and okr[: n // 4][a[: n // 4] > 0].mean() > 0.999
    # flags must fire on zero / signed-zero numerators, negative / special radicands
    idx = {v: i for i, v in enumerate(special)}
    grid = f[-special.size ** 2:].reshape(special.size, special.size)
    assert grid[idx[1.0], idx[0.0]] & 1 and grid[idx[1.0], idx[-0.0]] & 1  # a = +-0
    # grid[i, j] holds a = special[j], b = special[i]
    assert grid[idx[1.0], idx[-1.0]] & 2 and grid[idx[1.0], idx[np.inf]] & 2


@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (3, 8, 5), (2, 3, 11)])
def test_aos_soa_round_trip_matches_layout_enumerator(fvb, d, p, t):
    import torch

    lib = fvb.load_library()
    for haloed in (1, 0):
        m = p + 2 if haloed else p
        size = (d + 2) * t * m**d
        soa = torch.arange(size, dtype=torch.float64, device="cuda")
        aos = torch.empty_like(soa)
        back = torch.empty_like(soa)
        assert lib.fvb_soa_to_aos(d, p, t, haloed, soa.data_ptr(), aos.data_ptr(), None) == 0
        assert lib.fvb_aos_to_soa(d, p, t, haloed, aos.data_ptr(), back.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert torch.equal(back, soa)
        ref = oracle.soa_to_aos_patches(soa.cpu().numpy(), d, p, t, bool(haloed))
        assert np.array_equal(aos.cpu().numpy(), ref)


@pytest.mark.parametrize("realization", REALIZATIONS)
def test_constant_state_exact(fvb, realization):
    for d, q0 in ((2, (1.3, 0.26, -0.39, 3.25)), (3, (1.3, 0.26, -0.39, 0.13, 3.25))):
        p, t = 8, 9
        n, M, Mi = oracle.sizes(d, p, t)
        q = np.repeat(np.asarray(q0), t * M)
        out, red = _step(fvb, realization, d, p, t, q)
        assert out.tobytes() == np.repeat(np.asarray(q0), t * Mi).tobytes()
        params = fvb.EulerParameters()
        assert red == max(fvb.max_eigenvalue(q0, a, params) for a in range(d))


def test_flavours_agree_and_rerun_idempotent_at_scale(fvb):
    """C2 at full size (2D p=3, 100k patches): all flavours bit-identical,
    reruns bit-identical, sampled patches equal the oracle."""
    import torch

    d, p, t = 2, 3, 100_000
    shape = fvb.BatchShape(d, p, t)
    q = fvb.init_field_device(shape, 0)
    outs = {}
    for real in REALIZATIONS:
        outs[real] = _step(fvb, real, d, p, t, q_dev=q.tensor, lam_patch=True)
    again = _step(fvb, "patch-wise", d, p, t, q_dev=q.tensor, lam_patch=True)
    base = outs["patch-wise"]
    for real in REALIZATIONS[1:]:
        assert outs[real][0].tobytes() == base[0].tobytes()
        assert outs[real][1] == base[1]
        assert outs[real][2].tobytes() == base[2].tobytes()
    assert again[0].tobytes() == base[0].tobytes() and again[1] == base[1]
    assert base[1] == base[2].max()
    rng = np.random.default_rng(1)
    picks = np.sort(rng.choice(t, 64, replace=False))
    qs = q.as_array()[:, torch.as_tensor(picks, device="cuda"), :].contiguous().view(-1)
    ref_out, _, ref_lp = oracle.step_c(d, p, 64, qs.cpu().numpy(), lam_patch=True)
    got = base[0].reshape(d + 2, t, p * p)[:, picks, :].reshape(-1)
    assert got.tobytes() == ref_out.tobytes()
    assert base[2][picks].tobytes() == ref_lp.tobytes()


# C3 / C4 at full size: whole-batch oracle comparisons in test_gpu_fullsize.py


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16])
def test_3d_slab_sizes_match_oracle(fvb, p):
    """Every 3D patch size of the plane-walk kernel, a patch count that leaves
    slots with unequal work, reduction on and off."""
    d, t = 3, 37
    q = oracle.init_field_soa(d, p, t, 7)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    out, red, lp = _step(fvb, "patch-wise", d, p, t, q, lam_patch=True)
    assert out.tobytes() == ref_out.tobytes()
    assert red == ref_red
    assert lp.tobytes() == ref_lp.tobytes()
    out2, red2 = _step(fvb, "patch-wise", d, p, t, q, with_reduction=False)
    assert out2.tobytes() == ref_out.tobytes() and red2 is None


@pytest.mark.parametrize("d,p,t", [(2, 16, 1 << 18), (2, 3, 50_000), (3, 8, 20_000), (3, 6, 20_000), (3, 4, 30_000)])
def test_filtered_reduction_equals_exact(fvb, d, p, t):
    """Without per-patch maxima the fused kernels filter the eigenvalue
    reduction (Euler::lambda_below against the warp's running maximum).  The
    reduced eigenvalue must equal the exhaustive one bit for bit -- on the
    seeded field, on a field whose unique maximum sits in one late cell, and
    on a field of many near-ties (values just below / equal to the max)."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    q = fvb.init_field_device(shape, 5)
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_REDUCE_FILTER, 1):  # the filter on every kernel
        _filtered_cases(fvb, d, p, t, q)


def _filtered_cases(fvb, d, p, t, q):
    for variant in ("seeded", "late-peak", "ties"):
        qa = q.as_array().clone()  # [k][patch][lin]
        if variant == "late-peak":
            m = (p + 2) ** d
            lin = sum((p // 2 + 1) * (p + 2) ** i for i in range(d))  # an interior cell
            rho, m0 = float(qa[0, t - 3, lin]), float(qa[1, t - 3, lin])
            qa[1, t - 3, lin] = 3.0 * rho  # |u| = 3: the unique maximum ...
            qa[d + 1, t - 3, lin] += (9.0 * rho * rho - m0 * m0) / (2.0 * rho)  # ... same pressure
            assert lin < m
        elif variant == "ties":
            qa[:, :, :] = qa[:, :1, :1]  # one constant state everywhere ...
            qa[2, ::7, :] *= 1.0 + 2.0 ** -45  # ... a few patches perturbed in the last bits
        qv = qa.reshape(-1).contiguous()
        out_f, red_f = _step(fvb, "patch-wise", d, p, t, q_dev=qv)
        out_e, red_e, lp = _step(fvb, "patch-wise", d, p, t, q_dev=qv, lam_patch=True)
        assert out_f.tobytes() == out_e.tobytes()
        assert red_f == red_e == lp.max(), variant
        if variant == "late-peak":
            qs = qa[:, t - 3:t - 2, :].reshape(-1).cpu().numpy()
            _, ref_red = oracle.step_c(d, p, 1, qs)
            assert red_f == ref_red


def test_public_api_run_launch_copy_and_pooled(fvb):
    shape = fvb.BatchShape(2, 6, 16)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    q = oracle.init_field_soa(2, 6, 16, 260)
    ref_out, ref_red = oracle.step_c(2, 6, 16, q)
    arena = fvb.DeviceArena()
    for mode in (fvb.TransferMode.EXPLICIT_COPY, fvb.TransferMode.POOLED):
        for real in (fvb.Realization.PATCH_WISE, fvb.Realization.BATCHED,
                     fvb.Realization.TASK_GRAPH):
            sc = fvb.init_field(shape, 260)
            assert np.array_equal(sc.in_block, oracle.soa_to_aos_patches(q, 2, 6, 16, True))
            res = fvb.run_launch(plan, sc, fvb.Layout.SOA, real, mode,
                                 fvb.ReductionStrategy.GROUP_TREE, ctx, arena)
            assert res.reduced == ref_red
            assert np.concatenate(sc.outputs).tobytes() == \
                oracle.soa_to_aos_patches(ref_out, 2, 6, 16, False).tobytes()
            assert res.trace.executed_invocation_count == sum(res.trace.per_step_task_counts)
    pooled = fvb.DeviceArena()
    sc = fvb.init_field(shape, 260)
    for _ in range(5):
        fvb.run_launch(plan, sc, fvb.Layout.SOA, fvb.Realization.PATCH_WISE,
                       fvb.TransferMode.POOLED, fvb.ReductionStrategy.GROUP_TREE, ctx, pooled)
    assert pooled.allocation_count == 2 + 2 * shape.dim


def test_check_mode_raises_invalid_state(fvb):
    import torch

    shape = fvb.BatchShape(2, 4, 3)
    q = fvb.init_field_device(shape, 1)
    q.as_array()[0, 1, 7] = -1.0  # negative density in patch 1
    out = fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False)
    ctx = fvb.TimeStepContext(1e-3, 0.1, fvb.EulerParameters(), check=True)
    with pytest.raises(fvb.InvalidStateError):
        fvb.run_patchwise(fvb.build_plan(shape, True), q, out, None, ctx)


def test_workgroup_limit_semantics(fvb):
    import torch

    shape = fvb.BatchShape(3, 12, 1)  # 14^3 = 2744 > 1024
    q = fvb.init_field_device(shape, 2)
    out = fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False)
    ctx = fvb.default_context()
    plan = fvb.build_plan(shape, False)
    with pytest.raises(fvb.WorkgroupLimitError):
        fvb.run_patchwise(plan, q, out, None, ctx, workgroup_limit=1024)
    ref_out, _ = oracle.step_c(3, 12, 1, q.tensor.cpu().numpy(), with_reduction=False)
    # with the limit raised (as the reference allows) the fused plane walk runs it
    out.tensor.zero_()
    red, _ = fvb.run_patchwise(plan, q, out, None, ctx, workgroup_limit=2744)
    assert red is None and out.tensor.cpu().numpy().tobytes() == ref_out.tobytes()
    red, trace = fvb.run_batched(plan, q, out, None, ctx)
    assert red is None and trace.launch_count == 10
    assert out.tensor.cpu().numpy().tobytes() == ref_out.tobytes()
    # beyond the largest compiled plane walk (3D p = 16) the fused flavour refuses
    big = fvb.BatchShape(3, 20, 1)
    qb = fvb.init_field_device(big, 2)
    ob = fvb.DeviceFieldView(torch.zeros(big.output_size, dtype=torch.float64, device="cuda"), big, False)
    with pytest.raises(fvb.WorkgroupLimitError):
        fvb.run_patchwise(fvb.build_plan(big, False), qb, ob, None, ctx, workgroup_limit=1 << 20)


def test_graph_scratch_chunks_and_rebinding(fvb):
    import torch

    d, p, t = 2, 8, 50
    shape = fvb.BatchShape(d, p, t)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    scratch = fvb.GpuScratch(shape, fvb.Realization.TASK_GRAPH, chunks=4)
    for seed in (1, 2):  # second call rebinds the instantiated graph to new buffers
        q = fvb.init_field_device(shape, seed)
        out = fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64,
                                              device="cuda"), shape, False)
        red, trace = fvb.run_taskgraph(plan, q, out, scratch, ctx)
        ref_out, ref_red = oracle.step_c(d, p, t, q.tensor.cpu().numpy())
        assert out.tensor.cpu().numpy().tobytes() == ref_out.tobytes() and red == ref_red
        assert trace.launch_count == t * 8  # the reference's DAG node count (T*steps)
        assert trace.gpu_kernel_launches == 4 * 8  # 4 chunks x 8 step kernels
    assert scratch.graph_nodes() == 1 + 4 * 8
    scratch.close()


def test_rcp64h_scaling(fvb):
    """realx.cuh XScaled: fast_recip(2x) == 0.5*fast_recip(x) for every high
    mantissa over rho's certified exponent range [2^-250, 2^250) (and beyond)."""
    import torch

    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    assert fvb.load_library().fvb_probe_rcp_scaling(1023 - 300, 1023 + 300, bad.data_ptr(),
                                                    None) == 0
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


def _same_bits_nan_aware(a, b):
    """Byte equality, except that any NaN equals any NaN (NaN payloads are
    implementation-defined: x86 and CUDA produce different default NaNs)."""
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and a[~na].tobytes() == b[~nb].tobytes()


@pytest.mark.parametrize("d,p,t", [(2, 16, 3000), (2, 3, 4000), (2, 5, 999), (3, 8, 300), (3, 6, 500), (3, 4, 700)])
@pytest.mark.parametrize("realization", REALIZATIONS)
def test_degenerate_states_take_the_ieee_redo(fvb, d, p, t, realization):
    """Patches holding states outside the fast paths' certified range (tiny /
    huge magnitudes, -0 momentum, negative pressure, zero density) sit
    among ordinary ones: the fused kernels redo exactly those groups / patches
    in IEEE double and the whole batch still matches the oracle bit for bit
    (NaN-aware), eigenvalue included."""
    n = d + 2
    q = oracle.init_field_soa(d, p, t, 11).reshape(n, t, -1).copy()
    lin = sum((p // 2 + 1) * (p + 2) ** i for i in range(d))  # an interior cell
    q[0, 3, lin] = 1e-300                                      # tiny density
    q[1, 7, lin] = -0.0                                        # -0 momentum
    q[n - 1, 11, lin] = 1e-3                                   # negative pressure
    q[1, 13, :] *= 1e100                                       # huge momenta, whole patch
    q[:, 17, lin + 1] = 0.0                                    # zero state
    q[0, t - 1, 0] = 1e-80                                     # tiny density in a halo cell
    q = q.reshape(-1)
    ref_out, ref_red, ref_lp = oracle.step_c(d, p, t, q, lam_patch=True)
    out, red = _step(fvb, realization, d, p, t, q)
    assert _same_bits_nan_aware(out, ref_out)
    assert red == ref_red
    out2, red2, lp = _step(fvb, realization, d, p, t, q, lam_patch=True)
    assert _same_bits_nan_aware(out2, ref_out) and red2 == ref_red
    assert _same_bits_nan_aware(lp, ref_lp)


@pytest.mark.parametrize("d,p,t", [(2, 16, 4_200_000), (3, 8, 1_100_000)])
def test_large_batch_64bit_offsets(fvb, d, p, t):
    """Batches whose SoA offsets pass 2^32 (N*T*M > 4.3e9, the C5 per-GPU
    shard sizes): the fused kernel's last patches equal the oracle, and the
    field generator's jump-ahead agrees with the oracle there too."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    n, M, Mi = d + 2, (p + 2) ** d, p ** d
    assert n * t * M > 2**32
    q = fvb.init_field_device(shape, 3)
    out = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64, device="cuda"),
                              shape, False)
    ctx = fvb.default_context()
    lp = torch.empty(t, dtype=torch.float64, device="cuda")
    lam = fvb.step_async(fvb.Realization.PATCH_WISE, fvb.build_plan(shape, True), q, out, ctx,
                         lam_patch=lp)
    torch.cuda.synchronize()
    picks = torch.as_tensor([0, t // 2, t - 2, t - 1], device="cuda")
    qs = q.as_array()[:, picks, :].contiguous().view(-1).cpu().numpy()
    ref_out, _, ref_lp = oracle.step_c(d, p, len(picks), qs, lam_patch=True)
    got = out.tensor.view(n, t, Mi)[:, picks, :].contiguous().view(-1).cpu().numpy()
    assert got.tobytes() == ref_out.tobytes()
    assert lp[picks].cpu().numpy().tobytes() == ref_lp.tobytes()
    assert float(lam.item()) == float(lp.max().item())
    # jump-ahead: the last patch's input bits, drawn in pure Python from the
    # reference's LCG stream position (t-1)*M*N (bench.py:89-133)
    state = oracle.lcg_jump(3, (t - 1) * M * n)
    last = np.empty((n, M))
    for lin in range(M):
        draws = []
        for lo, hi in [(0.5, 2.0)] + [(-0.5, 0.5)] * d + [(0.5, 2.0)]:
            state = (state * oracle.LCG_A + oracle.LCG_C) & oracle.MASK64
            draws.append(lo + (hi - lo) * ((state >> 11) * 2.0**-53))
        rho, u, pr = draws[0], draws[1:1 + d], draws[1 + d]
        ke = u[0] * u[0] + u[1] * u[1]
        if d == 3:
            ke = ke + u[2] * u[2]
        last[0, lin] = rho
        for i in range(d):
            last[1 + i, lin] = rho * u[i]
        last[d + 1, lin] = pr / (1.4 - 1.0) + 0.5 * rho * ke
    assert q.as_array()[:, t - 1, :].contiguous().view(-1).cpu().numpy().tobytes() == last.tobytes()
    del q, out, lp
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p", [3, 5, 6, 7])
def test_partly_filled_warps_do_not_leak_into_the_reduction(fvb, p):
    """Patch sizes whose lanes do not fill a warp (32 % (p/C) != 0) leave
    lanes running on stand-in data.  After a high-eigenvalue step has left
    large values in shared memory, a low-eigenvalue field must still reduce
    to exactly the oracle's eigenvalue (filtered and exhaustive) -- stand-in
    lanes never feed tau, the running maximum or the redo vote."""
    import torch

    d, t = 2, 4099
    hot = oracle.init_field_soa(d, p, t, 9).reshape(d + 2, t, -1).copy()
    hot[1] *= 6.0  # large velocities -> large eigenvalues ...
    hot[d + 1] += 0.5 * (hot[1] ** 2 * (1 - 1 / 36.0)) / hot[0]  # ... at unchanged pressure
    hot = hot.reshape(-1)
    cold = oracle.init_field_soa(d, p, t, 10).reshape(d + 2, t, -1).copy()
    cold[1:d + 1] *= 0.01  # nearly at rest: small eigenvalues
    cold = cold.reshape(-1)
    _, red_hot = oracle.step_c(d, p, t, hot)
    ref_out, ref_red = oracle.step_c(d, p, t, cold)
    assert red_hot > 2 * ref_red
    for filt in (1, 0):
        with fvb._lib.tuning(fvb._lib.FVB_TUNE_REDUCE_FILTER, filt):
            _step(fvb, "patch-wise", d, p, t, hot)
            out, red = _step(fvb, "patch-wise", d, p, t, cold)
        assert red == ref_red, filt
        assert out.tobytes() == ref_out.tobytes()


@pytest.mark.parametrize("realization", REALIZATIONS)
@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (2, 3, 70), (3, 8, 21), (3, 5, 19), (2, 32, 5)])
def test_local_time_stepping_matches_per_patch_oracle(fvb, realization, d, p, t):
    """fvb_step_lts: every patch advances with its own dt; each patch's bytes,
    its eigenvalue and the batch maximum equal the oracle stepping that patch
    alone with that dt."""
    import torch

    n = d + 2
    q = oracle.init_field_soa(d, p, t, 17)
    rng = np.random.default_rng(5)
    dts = 1e-3 * rng.uniform(0.3, 1.7, t)
    dts[t // 2] = 2.0**-1010 * 0.1  # a dt/h outside the fast range: that patch's IEEE redo
    qa = q.reshape(n, t, -1)
    ref_out = np.empty((n, t, p**d))
    ref_lp = np.empty(t)
    for i in range(t):
        o, r = oracle.step_c(d, p, 1, np.ascontiguousarray(qa[:, i:i + 1, :]).reshape(-1), dt=dts[i], h=0.1)
        ref_out[:, i, :] = o.reshape(n, p**d)
        ref_lp[i] = r
    shape = fvb.BatchShape(d, p, t)
    inp = fvb.DeviceFieldView(torch.from_numpy(q).cuda(), shape, True)
    out = fvb.DeviceFieldView(torch.full((shape.output_size,), float("nan"), dtype=torch.float64,
                                         device="cuda"), shape, False)
    lp = torch.empty(t, dtype=torch.float64, device="cuda")
    ctx = fvb.default_context()
    for lam_patch in (None, lp):
        lam = fvb.step_async(fvb.Realization(realization), fvb.build_plan(shape, True), inp, out, ctx,
                             lam_patch=lam_patch, dt_patch=torch.from_numpy(dts).cuda())
        torch.cuda.synchronize()
        assert out.tensor.cpu().numpy().tobytes() == ref_out.reshape(-1).tobytes()
        assert float(lam.item()) == ref_lp.max()
    assert lp.cpu().numpy().tobytes() == ref_lp.tobytes()


@pytest.mark.parametrize("variant", [0, 8])
@pytest.mark.parametrize("p,t", [(16, 64), (16, 1), (16, 2), (16, 3), (16, 2001), (8, 4), (8, 37),
                                 (4, 9), (2, 17), (2, 15), (32, 3), (3, 40)])
@pytest.mark.parametrize("lam_patch", [False, True])
def test_pencil_launch_variants_match_oracle(fvb, variant, p, t, lam_patch):
    """Both 2D pencil launch shapes -- the TMA-streamed rows (0 = default;
    end-aligned groups, tensor-map halo columns), the cp.async ring (8) and batches
    smaller than one warp's group -- bit-identical to the oracle, with and
    without per-patch maxima (filtered vs exhaustive reduction)."""
    q = oracle.init_field_soa(2, p, t, 100 + p + t)
    ref_out, ref_red, ref_lp = oracle.step_c(2, p, t, q, lam_patch=True)
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_PENCIL_VARIANT, variant):
        res = _step(fvb, "patch-wise", 2, p, t, q, lam_patch=lam_patch)
    assert res[0].tobytes() == ref_out.tobytes()
    assert res[1].hex() == ref_red.hex()
    if lam_patch:
        assert res[2].tobytes() == ref_lp.tobytes()


@pytest.mark.parametrize("p", [6, 8])
@pytest.mark.parametrize("variant", [0, 5])
@pytest.mark.parametrize("t", [1, 2, 3, 64, 257])
@pytest.mark.parametrize("filtered", [0, 1])
def test_slab_launch_variants_match_oracle(fvb, p, variant, t, filtered):
    """3D launch shapes -- p = 8: the one-warp tensor-map kernel (0) and the
    two-warp slot kernel (5); p = 6: the slot kernel -- bit-identical to
    the oracle with the filtered and the exhaustive reduction, with and
    without per-patch maxima."""
    q = oracle.init_field_soa(3, p, t, 300 + t)
    ref_out, ref_red, ref_lp = oracle.step_c(3, p, t, q, lam_patch=True)
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_SLAB_VARIANT, variant), \
            fvb._lib.tuning(fvb._lib.FVB_TUNE_REDUCE_FILTER, filtered):
        out, red = _step(fvb, "patch-wise", 3, p, t, q)
        out2, red2, lp = _step(fvb, "patch-wise", 3, p, t, q, lam_patch=True)
    assert out.tobytes() == ref_out.tobytes() and out2.tobytes() == ref_out.tobytes()
    assert red.hex() == ref_red.hex() and red2.hex() == ref_red.hex()
    assert lp.tobytes() == ref_lp.tobytes()


@pytest.mark.parametrize("realization", REALIZATIONS)
@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (2, 8, 9), (2, 3, 11), (3, 8, 5), (3, 6, 3), (3, 5, 4)])
def test_unaligned_batch_takes_the_fallback_bit_exact(fvb, d, p, t, realization):
    """A batch that starts 8 bytes past a 16-byte boundary cannot be described
    by a tensor map: the launcher must fall back (cp.async ring / slot
    kernel) and still return the oracle's bits."""
    import torch

    q = oracle.init_field_soa(d, p, t, 400 + t)
    ref_out, ref_red, _ = oracle.step_c(d, p, t, q, lam_patch=True)
    buf = torch.empty(q.size + 1, dtype=torch.float64, device="cuda")
    view = buf[1:]
    assert view.data_ptr() % 16 == 8
    view.copy_(torch.from_numpy(np.ascontiguousarray(q)))
    out, red = _step(fvb, realization, d, p, t, q_dev=view)
    assert out.tobytes() == ref_out.tobytes()
    assert red.hex() == ref_red.hex()


@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (3, 8, 5)])
def test_unaligned_output_bit_exact(fvb, d, p, t):
    """An output batch starting 8 bytes past a 16-byte boundary: every store
    of the fused kernels is a scalar 8-byte store."""
    import torch

    q = oracle.init_field_soa(d, p, t, 500 + t)
    ref_out, ref_red, _ = oracle.step_c(d, p, t, q, lam_patch=True)
    shape = fvb.BatchShape(d, p, t)
    inp = fvb.DeviceFieldView(torch.from_numpy(np.ascontiguousarray(q)).cuda(), shape, True)
    buf = torch.full((shape.output_size + 1,), float("nan"), dtype=torch.float64, device="cuda")
    out = fvb.DeviceFieldView(buf[1:], shape, False)
    assert out.tensor.data_ptr() % 16 == 8
    ctx = fvb.TimeStepContext(1e-3, 0.1, fvb.EulerParameters(1.4))
    lam = fvb.step_async(fvb.Realization("patch-wise"), fvb.build_plan(shape, True), inp, out, ctx)
    torch.cuda.synchronize()
    assert out.tensor.cpu().numpy().tobytes() == ref_out.tobytes()
    assert float(lam.item()).hex() == ref_red.hex()


@pytest.mark.parametrize("t", [2, 32, 34, 64, 1000, 4098])
@pytest.mark.parametrize("filtered", [-1, 0, 1])
def test_tile_kernel_p3_matches_oracle_and_pencil(fvb, t, filtered):
    """2D p=3 (C2's patch size): the two-warp thread-per-patch kernel
    (fused2d_tile.cuh, default for even batches) equals the oracle and the
    pencil kernel (FVB_TUNE_PENCIL_VARIANT=6) bit for bit -- full and partial
    32-patch groups, filtered / exhaustive reduction, per-patch maxima, and
    local time stepping (per-patch dt)."""
    import torch

    q = oracle.init_field_soa(2, 3, t, 500 + t)
    ref_out, ref_red, ref_lp = oracle.step_c(2, 3, t, q, lam_patch=True)
    with fvb._lib.tuning(fvb._lib.FVB_TUNE_REDUCE_FILTER, filtered):
        for variant in (0, 6):
            with fvb._lib.tuning(fvb._lib.FVB_TUNE_PENCIL_VARIANT, variant):
                out, red = _step(fvb, "patch-wise", 2, 3, t, q)
                out2, red2, lp = _step(fvb, "patch-wise", 2, 3, t, q, lam_patch=True)
            assert out.tobytes() == ref_out.tobytes() and out2.tobytes() == ref_out.tobytes(), variant
            assert red.hex() == ref_red.hex() and red2.hex() == ref_red.hex(), variant
            assert lp.tobytes() == ref_lp.tobytes(), variant
    # local time stepping: every patch its own dt, each equal to the oracle stepping it alone
    shape = fvb.BatchShape(2, 3, t)
    dts = torch.linspace(1e-4, 2e-3, t, dtype=torch.float64, device="cuda")
    inp = fvb.DeviceFieldView(torch.from_numpy(q).cuda(), shape, True)
    out = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64, device="cuda"), shape, False)
    lam = fvb.step_async(fvb.Realization.PATCH_WISE, fvb.build_plan(shape, True), inp, out,
                         fvb.default_context(), dt_patch=dts)
    torch.cuda.synchronize()
    got = out.tensor.cpu().numpy().reshape(4, t, 9)
    qs = q.reshape(4, t, 25)
    for i in sorted({0, 1, t // 2, t - 1}):
        r_out, _ = oracle.step_c(2, 3, 1, qs[:, i:i + 1, :].copy().reshape(-1), dt=float(dts[i]))
        assert got[:, i, :].tobytes() == r_out.reshape(4, 9).tobytes(), i
