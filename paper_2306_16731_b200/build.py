"""Build libfvb.so in-tree with nvcc for sm_100a.

    python -m paper_2306_16731_b200.build [--force]

Translation units (csrc/host.h explains the split) compile in parallel; the
fused 2D pencil kernel is compiled once per patch size (pencil.cu with
-DFVB_P=<p>), which keeps every NVVM module small.  --fmad=false keeps every
a*b+c a rounded multiply and a rounded add (bit parity with the numpy /
Python reference); -lineinfo maps ncu's source page to csrc/.  The .so lands
next to this file so it travels with the repo snapshot to the GPU box
(git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "_obj"
LIB = PKG / "libfvb.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC"]
# A/B builds: extra -D flags and another output (FVB_LIBRARY selects it at run time)
NVCC_FLAGS += os.environ.get("FVB_EXTRA_NVCC_FLAGS", "").split()
if os.environ.get("FVB_BUILD_OUT"):
    OBJ = Path(os.environ["FVB_BUILD_OUT"]) / "_obj"
    LIB = Path(os.environ["FVB_BUILD_OUT"]) / "libfvb.so"
PENCIL_SIZES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 32]  # = FVB_PENCIL_SIZES
SLAB_SIZES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16]  # = FVB_SLAB_SIZES (3D; even p: TMA planes, odd p: cp.async)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfvb.so")


def units() -> list[tuple[Path, list[str], Path]]:
    """(source, extra flags, object) for every translation unit."""
    out = [(CSRC / f"{name}.cu", [], OBJ / f"{name}.o")
           for name in ("fvb", "generic", "cascade", "misc")]
    out += [(CSRC / "xfer.cu", ["-Xcompiler", "-fopenmp"], OBJ / "xfer.o")]  # host-staged gather / scatter
    out += [(CSRC / "pencil.cu", [f"-DFVB_P={p}"], OBJ / f"pencil_p{p}.o") for p in PENCIL_SIZES]
    out += [(CSRC / "slab3d.cu", [f"-DFVB_P3={p}"], OBJ / f"slab3d_p{p}.o") for p in SLAB_SIZES]
    return out


HOSTPTR_SRC = CSRC / "hostptr.c"


def hostptr_path() -> Path:
    import sysconfig

    return PKG / ("_hostptr" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_hostptr(force: bool = False, verbose: bool = False) -> Path:
    """The pointer-table CPython extension (host C, gcc)."""
    import sysconfig

    import numpy

    out = hostptr_path()
    if not force and out.exists() and out.stat().st_mtime >= HOSTPTR_SRC.stat().st_mtime:
        return out
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
           "-I", numpy.get_include(), "-o", str(out), str(HOSTPTR_SRC)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


def headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [PKG.parent / "include" / "fvb.h"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in headers())


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(o.exists() and o.stat().st_mtime <= t and not _stale(o, s) for s, _, o in units())


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    build_hostptr(force, verbose)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    if not force and up_to_date():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    todo = [(s, f, o) for s, f, o in units() if force or _stale(o, s)]

    def compile_one(item):
        src, flags, obj = item
        cmd = [cc, *NVCC_FLAGS, *flags, "-c", "-o", str(obj), str(src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name} {flags}:\n{r.stderr}")
        return obj

    workers = jobs or max(1, min(len(todo), os.cpu_count() or 4))
    with ThreadPoolExecutor(workers) as pool:
        list(pool.map(compile_one, todo))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-Xcompiler", "-fopenmp", "-o", str(tmp), *[str(o) for _, _, o in units()]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
