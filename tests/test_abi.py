"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares with the ctypes signatures the package binds, and validates
arguments before touching the device (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "fvb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fvb_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2306_16731_b200 import _lib

    return _lib.load()


def test_header_symbols_all_exported_and_bound(lib):
    from paper_2306_16731_b200 import _lib

    names = header_functions()
    assert len(names) >= 17
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(names) == bound
    for name in names:
        assert hasattr(lib, name), name


def test_version_and_host_dt(lib):
    assert lib.fvb_version().decode().startswith("fvb ")
    assert lib.fvb_admissible_dt(2.0, 0.1, 0.5) == 0.5 * 0.1 / 2.0
    from paper_2306_16731_b200 import admissible_dt

    assert admissible_dt(2.6496686308461896, 0.1) == 0.5 * 0.1 / 2.6496686308461896


@pytest.mark.parametrize("dim,p,t", [(4, 4, 1), (2, 1, 1), (3, 4, 0)])
def test_step_rejects_bad_shapes_before_device_work(lib, dim, p, t):
    rc = lib.fvb_step(0, dim, p, t, None, None, 1e-3, 0.1, 1.4, 1, None, None, None)
    assert rc == -1
    assert lib.fvb_last_error()


def test_error_mapping():
    from paper_2306_16731_b200 import WorkgroupLimitError, _lib

    lib = _lib.load()
    lib.fvb_step(0, 5, 4, 1, None, None, 1e-3, 0.1, 1.4, 1, None, None, None)
    with pytest.raises(ValueError, match="dim must be 2 or 3"):
        _lib.check(-1)
    with pytest.raises(WorkgroupLimitError):
        _lib.check(-2)


def test_plan_create_rejects_unknown_flavour(lib):
    h = ctypes.c_void_p()
    assert lib.fvb_plan_create(7, 2, 4, 4, 1, ctypes.byref(h)) == -1
    assert b"flavour" in lib.fvb_last_error()


def test_library_is_sm100a_only():
    """The .so carries sm_100a SASS (cuobjdump), no PTX for JIT elsewhere."""
    import shutil
    import subprocess

    so = ROOT / "paper_2306_16731_b200" / "libfvb.so"
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run([tool, "--list-ptx", str(so)], capture_output=True, text=True).stdout
    assert ".ptx" not in ptx


def test_physics_selection_round_trip_and_validation(lib):
    """fvb_set_physics / fvb_get_physics (csrc/physics.cuh): the two compiled
    policies are selectable, anything else is rejected (no device work)."""
    from paper_2306_16731_b200 import _lib

    v = ctypes.c_int()
    assert lib.fvb_get_physics(ctypes.byref(v)) == 0
    assert v.value == _lib.FVB_PHYSICS_EULER
    with _lib.physics(_lib.FVB_PHYSICS_EULER_PLAIN):
        assert lib.fvb_get_physics(ctypes.byref(v)) == 0 and v.value == _lib.FVB_PHYSICS_EULER_PLAIN
    assert lib.fvb_get_physics(ctypes.byref(v)) == 0 and v.value == _lib.FVB_PHYSICS_EULER
    assert lib.fvb_set_physics(7) == -1 and b"physics" in lib.fvb_last_error()
    assert lib.fvb_get_physics(None) == -1
