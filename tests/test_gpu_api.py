"""GPU tests of the public API around the step: reference-schema sweeps and
CSV, trace invariants, the streamed host path, the sharded driver (1 rank).
Mirrors pkg/tests/test_acceptance.py (benchmark-protocol replica, trace
invariants, memory-mode counters) for the GPU realisations."""

import csv

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fvb(cuda):
    import paper_2306_16731_b200 as pkg

    pkg.load_library()
    return pkg


def test_sweep_csv_schema_and_normalisation(fvb, tmp_path):
    from paper_2306_16731_b200 import sweep

    configs = [sweep.BenchConfig(dim=2, patch_size=p, patch_count=t, realization=r, samples=3,
                                 with_reduction=wr)
               for p in (4, 8) for t in (1, 64) for wr in (True, False)
               for r in (fvb.Realization.PATCH_WISE, fvb.Realization.BATCHED,
                         fvb.Realization.TASK_GRAPH)]
    records = sweep.run_sweep(configs)
    assert [r.config.sort_key for r in records] == sorted(c.sort_key for c in configs)
    path = tmp_path / "sweep.csv"
    sweep.emit_csv(records, str(path))
    rows = list(csv.DictReader(open(path, newline="")))
    assert list(rows[0]) == sweep.CSV_HEADER and len(rows) == len(configs)
    for row in rows:
        total = float(row["mean_total_s"])
        vol = int(row["T"]) * int(row["p"]) ** int(row["dim"])
        assert float(row["time_per_volume_update_s"]) == total / vol
        assert float(row["time_per_unknown_update_s"]) == total / (vol * (int(row["dim"]) + 2))
        assert float(row["mean_compute_s"]) <= total
        if row["with_reduction"] == "true":
            q = oracle.init_field_soa(2, int(row["p"]), int(row["T"]), 0)
            assert float(row["reduced_eigenvalue"]) == oracle.step_c(2, int(row["p"]),
                                                                     int(row["T"]), q)[1]
        else:
            assert float(row["reduced_eigenvalue"]) == 0.0


@pytest.mark.parametrize("d,with_reduction", [(2, False), (2, True), (3, False), (3, True)])
def test_trace_invariants(fvb, d, with_reduction):
    import torch

    t = 2
    shape = fvb.BatchShape(d, 4, t)
    steps = 1 + 3 * d + (1 if with_reduction else 0)
    plan = fvb.build_plan(shape, with_reduction)
    q = fvb.init_field_device(shape, 3)
    ctx = fvb.default_context()

    def out():
        return fvb.DeviceFieldView(torch.zeros(shape.output_size, dtype=torch.float64,
                                               device="cuda"), shape, False)

    assert fvb.run_batched(plan, q, out(), None, ctx)[1].global_sync_count == steps
    tr = fvb.run_patchwise(plan, q, out(), None, ctx)[1]
    assert tr.global_sync_count == 1 and tr.launch_count == 1
    scratch = fvb.GpuScratch(shape, fvb.Realization.TASK_GRAPH, chunks=t)
    tr = fvb.run_taskgraph(plan, q, out(), scratch, ctx)[1]
    assert tr.launch_count == t * steps  # one node chain per patch, like the reference
    assert scratch.graph_nodes() == t * steps + (1 if with_reduction else 0)
    counts = [r.range_size * t for r in plan.steps]
    assert tr.per_step_task_counts == counts and tr.executed_invocation_count == sum(counts)


def test_streamed_step_matches_oracle(fvb):
    from paper_2306_16731_b200.pipeline import StreamedStep

    shape = fvb.BatchShape(2, 16, 1000)
    sc = fvb.init_field(shape, 11, pinned=True)
    ctx = fvb.default_context()
    red = StreamedStep(shape, chunks=7).run_scattered(sc, ctx)
    q = oracle.init_field_soa(2, 16, 1000, 11)
    ref_out, ref_red = oracle.step_c(2, 16, 1000, q)
    assert red == ref_red
    assert sc.out_block.tobytes() == oracle.soa_to_aos_patches(ref_out, 2, 16, 1000, False).tobytes()


def test_sharded_step_single_rank_equals_whole(fvb):
    from paper_2306_16731_b200.distributed import ShardedStep

    ctx = fvb.default_context()
    total = 37
    lams = []
    for world in (1, 2, 3):
        for rank in range(world):  # sequential "virtual ranks" on one device, max-combined
            s = ShardedStep(2, 8, total, rank, world, ctx, seed=5)
            lams.append((world, float(s.step().item())))
    q = oracle.init_field_soa(2, 8, total, 5)
    ref = oracle.step_c(2, 8, total, q)[1]
    for world in (1, 2, 3):
        assert max(l for w, l in lams if w == world) == ref


def test_pooled_counter_and_copy_counter(fvb):
    shape = fvb.BatchShape(2, 4, 2)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    base = fvb.init_field(shape, 4)
    pooled = fvb.DeviceArena()
    for _ in range(5):
        fvb.run_launch(plan, base, fvb.Layout.SOA, fvb.Realization.BATCHED,
                       fvb.TransferMode.POOLED, fvb.ReductionStrategy.GROUP_TREE, ctx, pooled)
    assert pooled.allocation_count == 2 + 2 * shape.dim  # input, output, d flux + d wave speed
    copy = fvb.DeviceArena()
    for i in range(3):
        fvb.run_launch(plan, base, fvb.Layout.SOA, fvb.Realization.BATCHED,
                       fvb.TransferMode.EXPLICIT_COPY, fvb.ReductionStrategy.GROUP_TREE, ctx, copy)
        assert copy.allocation_count == (2 + 2 * shape.dim) * (i + 1)
    dev = fvb.DevicePatchSet(shape, fvb.init_field_device(shape, 4),
                             fvb.DeviceFieldView(__import__("torch").zeros(
                                 shape.output_size, dtype=__import__("torch").float64,
                                 device="cuda"), shape, False))
    res = fvb.run_launch(plan, dev, fvb.Layout.SOA, fvb.Realization.PATCH_WISE,
                         fvb.TransferMode.SHARED, fvb.ReductionStrategy.GROUP_TREE, ctx,
                         fvb.DeviceArena())
    assert res.transfer_s == 0.0
    q = oracle.init_field_soa(2, 4, 2, 4)
    assert res.reduced == oracle.step_c(2, 4, 2, q)[1]


@pytest.mark.parametrize("d,p,grid", [(2, 16, (4, 3)), (2, 5, (3, 2)), (3, 4, (2, 3, 2))])
def test_multistep_simulation_matches_oracle(fvb, d, p, grid):
    """f2: step -> dt = cfl*h/lambda -> periodic halo refresh, three steps,
    bit-exact against the oracle step + numpy halo refresh."""
    from paper_2306_16731_b200.simulation import PatchGridSimulation

    sim = PatchGridSimulation(d, p, grid, seed=3, dt0=1e-3)
    t = int(np.prod(grid))
    q = oracle.init_field_soa(d, p, t, 3)
    dt = 1e-3
    for _ in range(3):
        out, red = oracle.step_c(d, p, t, q, dt=dt, h=0.1)
        q = oracle.refresh_halos_soa(d, p, grid, out)
        dt_gpu = sim.step()
        dt = 0.5 * 0.1 / red
        assert dt_gpu == dt
        assert sim.out.tensor.cpu().numpy().tobytes() == out.tobytes()
        assert sim.inp.tensor.cpu().numpy().tobytes() == q.tobytes()


@pytest.mark.parametrize("d,p,grid", [(2, 16, (8, 6)), (3, 8, (3, 2, 2)), (2, 5, (4, 3))])
def test_device_dt_steps_and_cuda_graph_match_host_dt(fvb, d, p, grid):
    """f2 without host synchronisation: dt kept in HBM (fvb_step_dt +
    fvb_admissible_dt_dev), the same steps captured as one CUDA graph and
    replayed -- bit-identical to the host-dt loop and to the oracle."""
    from paper_2306_16731_b200.simulation import PatchGridSimulation

    t = int(np.prod(grid))
    host = PatchGridSimulation(d, p, grid, seed=5, dt0=1e-3)
    dev = PatchGridSimulation(d, p, grid, seed=5, dt0=1e-3)
    gr = PatchGridSimulation(d, p, grid, seed=5, dt0=1e-3)
    q = oracle.init_field_soa(d, p, t, 5)
    dt, time = 1e-3, 0.0
    dts = []
    for _ in range(6):  # the oracle's loop
        out, red = oracle.step_c(d, p, t, q, dt=dt, h=0.1)
        q = oracle.refresh_halos_soa(d, p, grid, out)
        time += dt
        dt = 0.5 * 0.1 / red
        dts.append(dt)
    for _ in range(6):
        host.step()
    dev.run_device(6)
    gr.capture(5)  # one eager step, then 5 captured
    gr.replay()
    for sim in (host, dev, gr):
        dt_s, time_s = sim.sync_host() if sim is not host else (host.dt, host.time)
        assert dt_s == dts[-1] and time_s == time
        assert sim.out.tensor.cpu().numpy().tobytes() == out.tobytes()
        assert sim.inp.tensor.cpu().numpy().tobytes() == q.tobytes()


@pytest.mark.parametrize("realization", ["patch-wise", "batched", "task-graph"])
@pytest.mark.parametrize("d,p", [(2, 16), (3, 8), (2, 5)])
def test_device_dt_every_flavour(fvb, realization, d, p):
    """fvb_step_dt (dt read on the device) equals the host-dt step bit for bit
    in every flavour, and a changed device dt is picked up by a cached plan /
    instantiated CUDA graph without rebuilding."""
    import torch

    t = 37
    shape = fvb.BatchShape(d, p, t)
    q = fvb.init_field_device(shape, 4)
    plan = fvb.build_plan(shape, True)
    real = fvb.Realization(realization)
    dt_dev = torch.empty(1, dtype=torch.float64, device="cuda")
    for dt in (1e-3, 3.7e-4):
        ctx = fvb.TimeStepContext(dt, 0.1, fvb.EulerParameters(1.4))
        o_host = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64,
                                                 device="cuda"), shape, False)
        o_dev = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64,
                                                device="cuda"), shape, False)
        lam_h = fvb.step_async(real, plan, q, o_host, ctx)
        dt_dev.fill_(dt)
        lam_d = fvb.step_async(real, plan, q, o_dev, ctx, dt_dev=dt_dev)
        torch.cuda.synchronize()
        assert torch.equal(o_host.tensor, o_dev.tensor)
        assert float(lam_h.item()) == float(lam_d.item())
        ref_out, ref_red = oracle.step_c(d, p, t, q.tensor.cpu().numpy(), dt=dt, h=0.1)
        assert o_dev.tensor.cpu().numpy().tobytes() == ref_out.tobytes()
        assert float(lam_d.item()) == ref_red


@pytest.mark.parametrize("name", ["2d_p3_t5_soa", "3d_p2_t3_aosoa", "2d_p4_t2_aos"])
def test_load_batch_step_and_dump_round_trip(fvb, name, tmp_path):
    """A batch file the reference wrote (dump_batch) loads straight into HBM
    in its layout; stepping the loaded input gives the file's golden output;
    dump_batch writes the same bytes back."""
    import torch

    from golden_cases import GOLDEN

    path = GOLDEN / f"batch_{name}.bin"
    batch = fvb.load_batch(path)
    want = batch.output.tensor.clone()
    plan = fvb.build_plan(batch.shape, True)
    for real in (fvb.Realization.PATCH_WISE, fvb.Realization.BATCHED, fvb.Realization.TASK_GRAPH):
        batch.output.tensor.fill_(float("nan"))
        fvb.step_async(real, plan, batch.input, batch.output, fvb.default_context())
        torch.cuda.synchronize()
        assert torch.equal(batch.output.tensor, want), real
    out = tmp_path / "dump.bin"
    fvb.dump_batch(batch, out)
    assert out.read_bytes() == path.read_bytes()


def test_sweep_verify_mode_passes_and_names_the_first_mismatch(fvb, monkeypatch):
    """run_sweep(verify=True) (bench.py:271-374): every realisation / transfer
    mode / layout matches the golden run (cascade kernels, hook-free physics,
    SHARED AoS, check=True); a corrupted trial raises VerifyError naming the
    patch and offset."""
    from paper_2306_16731_b200 import sweep

    configs = [sweep.BenchConfig(dim=d, patch_size=p, patch_count=t, realization=r, transfer_mode=m,
                                 layout=lay, samples=1)
               for d, p, t in ((2, 4, 6), (3, 3, 2)) for r in (fvb.Realization.PATCH_WISE,
                                                               fvb.Realization.TASK_GRAPH)
               for m in fvb.TransferMode for lay in (fvb.Layout.SOA, fvb.Layout.AOS)]
    assert len(sweep.run_sweep(configs, verify=True)) == len(configs)

    real_launch = sweep.run_launch

    def corrupting(plan, scattered, layout, realization, *args, **kw):
        res = real_launch(plan, scattered, layout, realization, *args, **kw)
        if realization is fvb.Realization.PATCH_WISE:
            scattered.outputs[1][3] += 1.0
        return res

    monkeypatch.setattr(sweep, "run_launch", corrupting)
    with pytest.raises(fvb.VerifyError, match="patch 1 offset 3"):
        sweep.run_sweep([sweep.BenchConfig(dim=2, patch_size=4, patch_count=3, samples=1)], verify=True)


@pytest.mark.parametrize("flavour", ["FVB_FUSED", "FVB_CASCADE", "FVB_GRAPH"])
def test_per_thread_default_streams_do_not_share_state(fvb, flavour):
    """cudaStreamPerThread is one handle for one stream per host thread: the
    library's stream-keyed state -- the fused flavour's self-resetting
    reduction slot, the cached plans' scratch of the cascade / graph flavours
    -- must not be shared between threads whose launches overlap.  Two host
    threads launch on it (ctypes releases the GIL), each with its own batch;
    every eigenvalue and the final output must be its batch's."""
    import threading

    import torch

    from paper_2306_16731_b200 import _lib

    lib = fvb.load_library()
    fl = getattr(_lib, flavour)
    per_thread = 2  # cudaStreamPerThread
    # fused: small launches, two of them run side by side; cascade / graph:
    # launches long enough that both threads' stage kernels queue up and interleave
    shape = fvb.BatchShape(2, 16, 256 if flavour == "FVB_FUSED" else 20_000)
    ctx = fvb.default_context()
    qs = [fvb.init_field_device(shape, seed) for seed in (1, 2)]
    expect = []
    for q in qs:
        ref = torch.zeros(1, dtype=torch.float64, device="cuda")
        out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
        _lib.check(lib.fvb_step(_lib.FVB_FUSED, 2, 16, shape.patch_count, q.data_ptr(), out.data_ptr(), ctx.dt,
                                ctx.h, ctx.params.gamma, 1, ref.data_ptr(), None, None))
        torch.cuda.synchronize()
        expect.append((float(ref.item()), out.cpu()))
    assert expect[0][0] != expect[1][0]
    errors = []
    n = 200 if flavour == "FVB_FUSED" else 30

    def worker(i):
        try:
            out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
            lams = torch.zeros(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            for it in range(n):
                _lib.check(lib.fvb_step(fl, 2, 16, shape.patch_count, qs[i].data_ptr(), out.data_ptr(),
                                        ctx.dt, ctx.h, ctx.params.gamma, 1, lams[it:].data_ptr(), None, per_thread))
            torch.cuda.synchronize()
            got = lams.cpu().numpy()
            if not (got == expect[i][0]).all():
                errors.append((i, "eigenvalue", got))
            if not torch.equal(out.cpu(), expect[i][1]):
                errors.append((i, "output"))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((i, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in (0, 1)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    lib.fvb_release_all()
    assert not errors, errors


def test_overlapping_or_cross_device_views_are_rejected(fvb):
    """The step never writes its input (test_memory.py:170-178): an output
    view overlapping the input batch is refused before anything launches."""
    import torch

    shape = fvb.BatchShape(2, 4, 8)
    buf = torch.zeros(shape.input_size + shape.output_size, dtype=torch.float64, device="cuda")
    inp = fvb.DeviceFieldView(buf[:shape.input_size], shape, True)
    plan = fvb.build_plan(shape, True)
    ctx = fvb.default_context()
    bad = fvb.DeviceFieldView(buf[shape.input_size - 8:shape.input_size - 8 + shape.output_size], shape, False)
    with pytest.raises(ValueError, match="overlap"):
        fvb.step_async(fvb.Realization.PATCH_WISE, plan, inp, bad, ctx)
    good = fvb.DeviceFieldView(buf[shape.input_size:], shape, False)
    fvb.step_async(fvb.Realization.PATCH_WISE, plan, inp, good, ctx)
    torch.cuda.synchronize()


@pytest.mark.parametrize("own_plan", [False, True])
@pytest.mark.parametrize("realization", ["patch-wise", "batched", "task-graph"])
@pytest.mark.parametrize("d,p,t", [(2, 16, 37), (3, 8, 9), (2, 3, 70)])
def test_step_captured_in_a_user_cuda_graph(fvb, realization, d, p, t, own_plan):
    """A user capturing step_async into their own CUDA graph (torch.cuda.graph)
    and replaying it -- also after the inputs changed in place -- gets the
    eager step's bytes and eigenvalue: the fused flavour binds no stream-keyed
    reduction slot while captured, the cascade / graph flavours' cached plans
    capture their kernels (or instantiated graph) as nodes."""
    import torch

    shape = fvb.BatchShape(d, p, t)
    ctx = fvb.default_context()
    plan = fvb.build_plan(shape, True)
    real = fvb.Realization(realization)
    q = fvb.init_field_device(shape, 21)
    out = fvb.DeviceFieldView(torch.empty(shape.output_size, dtype=torch.float64, device="cuda"), shape, False)
    lam = torch.zeros(1, dtype=torch.float64, device="cuda")
    # own_plan: a caller-owned plan (GpuScratch) first used inside the capture
    # -- its task graph is instantiated there
    scratch = fvb.GpuScratch(shape, real) if own_plan and realization != "patch-wise" else None
    if scratch is None:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm: plans, slots, tensor-map encoders
            fvb.step_async(real, plan, q, out, ctx, lam=lam)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fvb.step_async(real, plan, q, out, ctx, lam=lam, scratch=scratch)
    for seed in (21, 22):
        q.tensor.copy_(fvb.init_field_device(shape, seed).tensor)
        out.tensor.fill_(float("nan"))
        lam.fill_(-1.0)
        g.replay()
        torch.cuda.synchronize()
        ref_out, ref_red = oracle.step_c(d, p, t, q.tensor.cpu().numpy())
        assert out.tensor.cpu().numpy().tobytes() == ref_out.tobytes(), (realization, seed)
        assert float(lam.item()) == ref_red, (realization, seed)
