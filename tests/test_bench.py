"""The bench.py contract: one JSON line with the driver's keys, for both arms,
at N = 1 and under torchrun (N = 2; on one GPU the ranks share the device
through bench.py's FVB_BENCH_DEVICE / FVB_BENCH_BACKEND test scaffolding)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, env=None, nproc=1, timeout=900):
    cmd = [sys.executable]
    if nproc > 1:
        cmd += ["-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000)]
    cmd += [str(ROOT / "bench.py")] + args + (["--gpus", str(nproc)] if nproc > 1 else [])
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def _check_base(d, n):
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == n and d["value"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["dtype"] == "f64"
    assert "workload" in d["config"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= d["e2e"].keys()


@pytest.mark.parametrize("nproc", [1, 2])
def test_reference_arm_prints_one_line(nproc):
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--patches", "256",
              "--no-extras"], nproc=nproc)
    _check_base(d, nproc)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_flag_reexecs_under_torchrun_and_rejects_mismatch():
    """--gpus N without torchrun re-launches N ranks (rank 0 prints); a
    WORLD_SIZE that disagrees with --gpus is refused."""
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--patches", "128",
              "--no-extras", "--gpus", "2"])
    assert d["n_gpus"] == 2
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--patches", "64", "--no-extras"], cwd=ROOT, capture_output=True, text=True,
                       env=dict(os.environ, WORLD_SIZE="2", RANK="0"), timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


FAST = ["--patches", "4096", "--steps", "3", "--warmup", "3", "--warmup-seconds", "0",
        "--cpu-seconds", "0.5", "--e2e-steps", "2", "--e2e-chunk-patches", "1000", "--no-extras"]


@pytest.mark.gpu
def test_gpu_arm_contract(cuda):
    d = _run(FAST)
    _check_base(d, 1)
    assert d["gpu_launches"] >= d["steps"]
    x = d["exhaustive"]
    assert x["value"] > 0 and 0 < x["roofline_frac"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] == rf["achieved"] / rf["peak"]
    assert rf["algorithmic_bytes_per_launch"] == 4096 * 8 * 4 * (18 * 18 + 16 * 16)
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["kind"] == "port" and cb["cores"] >= 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 4096 * 8 * 4 * 18 * 18 and e["value"] > 0
    assert "run_launch" in e["path"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["reduced_eigenvalue"] > 0


@pytest.mark.gpu
def test_gpu_arm_two_ranks_share_the_eigenvalue(cuda):
    """N = 2 ranks (one GPU, gloo): whole-job value over both shards, the
    all-reduced eigenvalue equal to the single-rank run over both shards."""
    env = {"FVB_BENCH_DEVICE": "0", "FVB_BENCH_BACKEND": "gloo"}
    d2 = _run(FAST + ["--no-cpu"], env=env, nproc=2)
    _check_base(d2, 2)
    assert d2["config"]["total_patches"] == 2 * 4096
    d1 = _run(["--patches", "8192", "--steps", "3", "--warmup", "3", "--warmup-seconds", "0",
               "--no-cpu", "--no-e2e"])
    assert d2["reduced_eigenvalue"] == d1["reduced_eigenvalue"]
