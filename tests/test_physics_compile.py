"""The microkernel contract is N-generic (csrc/physics.cuh): a user policy
with a different state length -- Euler plus an advected tracer, N = d + 3,
stated as plain double functions without hooks -- instantiates every fused
and cascade kernel template (tests/physics/tracer_policy.cu).  Compile-only
(no GPU): nvcc cross-compiles for sm_100a here."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    return None


@pytest.mark.skipif(_nvcc() is None, reason="needs nvcc")
def test_tracer_policy_instantiates_every_kernel_family(tmp_path):
    obj = tmp_path / "tracer.o"
    r = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                        "-std=c++17", "-c", "-o", str(obj), str(ROOT / "tests" / "physics" / "tracer_policy.cu")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    syms = subprocess.run(["cuobjdump", "--dump-resource-usage", str(obj)], capture_output=True,
                          text=True).stdout
    for kernel in ("fused2d_pencil_kernel", "fused2d_pencil_tma_kernel", "fused2d_tile_kernel",
                   "fused3d_warp_kernel", "fused3d_slab_kernel", "fused_generic_kernel",
                   "cascade_flux_kernel", "cascade_acc_kernel", "cascade_reduce_kernel"):
        assert kernel in syms and "EulerTracer" in syms, kernel
