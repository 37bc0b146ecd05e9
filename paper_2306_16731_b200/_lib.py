"""ctypes binding of libfvb.so (include/fvb.h).

The product path has exactly one implementation: the CUDA library.  If the
library is missing or cannot be loaded this module raises -- there is no CPU
fallback.  Error codes map onto the reference's exception classes
(include/fvb.h "Error codes").
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from .errors import InvalidStateError, WorkgroupLimitError

import os

# FVB_LIBRARY: an alternative build of the same ABI (A/B experiments)
LIB_PATH = Path(os.environ.get("FVB_LIBRARY") or Path(__file__).resolve().parent / "libfvb.so")

FVB_FUSED, FVB_CASCADE, FVB_GRAPH = 0, 1, 2
FVB_LAYOUT_AOS, FVB_LAYOUT_SOA, FVB_LAYOUT_AOSOA = 0, 1, 2
FVB_TUNE_PENCIL_VARIANT, FVB_TUNE_SLAB_VARIANT, FVB_TUNE_REDUCE_FILTER = 0, 1, 2
FVB_PHYSICS_EULER, FVB_PHYSICS_EULER_PLAIN = 0, 1
FVB_OK, FVB_EINVAL, FVB_ELIMIT, FVB_ECUDA, FVB_EINVALID_STATE = 0, -1, -2, -3, -4

_c_int, _c_i64, _c_u64, _c_d, _c_p = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_double, ctypes.c_void_p)

# (name, restype, argtypes) for every symbol include/fvb.h declares
SIGNATURES = [
    ("fvb_version", ctypes.c_char_p, []),
    ("fvb_last_error", ctypes.c_char_p, []),
    ("fvb_step", _c_int, [_c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_d, _c_d, _c_d, _c_int,
                          _c_p, _c_p, _c_p]),
    ("fvb_step_layout", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_d, _c_d, _c_d,
                                 _c_int, _c_p, _c_p, _c_p]),
    ("fvb_step_dt", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d,
                             _c_int, _c_p, _c_p, _c_p]),
    ("fvb_admissible_dt_dev", _c_int, [_c_p, _c_d, _c_d, _c_p, _c_p]),
    ("fvb_step_lts", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d,
                              _c_int, _c_p, _c_p, _c_p]),
    ("fvb_plan_set_layout", _c_int, [_c_p, _c_int]),
    ("fvb_relayout", _c_int, [_c_int, _c_int, _c_i64, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_plan_create", _c_int, [_c_int, _c_int, _c_int, _c_i64, _c_int, ctypes.POINTER(_c_p)]),
    ("fvb_plan_execute", _c_int, [_c_p, _c_p, _c_p, _c_d, _c_d, _c_d, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_plan_graph_nodes", _c_int, [_c_p, ctypes.POINTER(_c_i64)]),
    ("fvb_plan_kernel_launches", _c_int, [_c_p, _c_int, ctypes.POINTER(_c_i64)]),
    ("fvb_plan_destroy", _c_int, [_c_p]),
    ("fvb_release_all", _c_int, []),
    ("fvb_fused_limit", _c_int, [_c_int, ctypes.POINTER(_c_int)]),
    ("fvb_fused_smem_bytes", _c_int, [_c_int, _c_int, ctypes.POINTER(_c_i64)]),
    ("fvb_set_tuning", _c_int, [_c_int, _c_int]),
    ("fvb_get_tuning", _c_int, [_c_int, ctypes.POINTER(_c_int)]),
    ("fvb_set_physics", _c_int, [_c_int]),
    ("fvb_get_physics", _c_int, [ctypes.POINTER(_c_int)]),
    ("fvb_init_field", _c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_u64, _c_d, _c_p, _c_p]),
    ("fvb_aos_to_soa", _c_int, [_c_int, _c_int, _c_i64, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_soa_to_aos", _c_int, [_c_int, _c_int, _c_i64, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_eval_microkernels", _c_int, [_c_int, _c_i64, _c_int, _c_d, _c_int, _c_p, _c_p, _c_p, _c_p]),
    ("fvb_probe_fastmath", _c_int, [_c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    ("fvb_probe_rcp_scaling", _c_int, [_c_int, _c_int, _c_p, _c_p]),
    ("fvb_check_admissible", _c_int, [_c_int, _c_int, _c_i64, _c_int, _c_d, _c_p, _c_p, _c_p]),
    ("fvb_refresh_halos", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_admissible_dt", _c_d, [_c_d, _c_d, _c_d]),
    ("fvb_check_admissible_ex", _c_int, [_c_int, _c_int, _c_i64, _c_int, _c_int, _c_d, _c_p, _c_p, _c_p,
                                         _c_p]),
    ("fvb_host_pin", _c_int, [_c_p, _c_i64, _c_i64, ctypes.POINTER(_c_p)]),
    ("fvb_host_note_pinned", _c_int, [_c_p, _c_i64, ctypes.POINTER(_c_p)]),
    ("fvb_host_unpin", _c_int, [_c_p]),
    ("fvb_host_accessible", _c_int, [_c_p, _c_i64, _c_i64, ctypes.POINTER(_c_i64)]),
    ("fvb_gather_table", _c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_p, _c_int, _c_p, _c_p]),
    ("fvb_scatter_table", _c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_step_table", _c_int, [_c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_d, _c_d, _c_d, _c_int,
                                _c_p, _c_p, _c_p]),
    ("fvb_step_range", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_d,
                                _c_d, _c_d, _c_int, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_plan_execute_ex", _c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_int, _c_d, _c_d,
                                     _c_d, _c_int, _c_p, _c_p, _c_p]),
    ("fvb_scratch_doubles", _c_int, [_c_int, _c_int, _c_i64, ctypes.POINTER(_c_i64),
                                     ctypes.POINTER(_c_i64)]),
    ("fvb_plan_create_ext", _c_int, [_c_int, _c_int, _c_int, _c_i64, _c_int, _c_p, _c_p,
                                     ctypes.POINTER(_c_p)]),
    ("fvb_launch_table", _c_int, [_c_int, _c_int, _c_int, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                                  _c_d, _c_d, _c_d, _c_int, _c_p, _c_i64, ctypes.POINTER(_c_d),
                                  ctypes.POINTER(_c_d), _c_p]),
]

_lib: ctypes.CDLL | None = None


class FvbError(RuntimeError):
    """A CUDA-side failure reported by libfvb (FVB_ECUDA)."""


def load() -> ctypes.CDLL:
    """Load libfvb.so (building it first if the toolkit is present)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        from . import build as _build

        _build.build()
    if not LIB_PATH.exists():
        raise ImportError(f"libfvb.so not found at {LIB_PATH}; run python -m paper_2306_16731_b200.build")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Raise the reference-equivalent exception for a non-zero return code."""
    if rc == FVB_OK:
        return
    msg = load().fvb_last_error().decode(errors="replace")
    if rc == FVB_EINVAL:
        raise ValueError(msg)
    if rc == FVB_ELIMIT:
        raise WorkgroupLimitError(msg)
    if rc == FVB_EINVALID_STATE:
        raise InvalidStateError(msg)
    raise FvbError(msg or f"libfvb error {rc}")


class tuning:
    """Context manager: set a launch-tuning knob (fvb_set_tuning) for a block.

    with tuning(FVB_TUNE_REDUCE_FILTER, 1): ...
    """

    def __init__(self, key: int, value: int) -> None:
        self.key, self.value = key, value

    def __enter__(self):
        lib = load()
        old = _c_int()
        check(lib.fvb_get_tuning(self.key, ctypes.byref(old)))
        self.old = old.value
        check(lib.fvb_set_tuning(self.key, self.value))
        return self

    def __exit__(self, *exc):
        check(load().fvb_set_tuning(self.key, self.old))


def current_physics() -> int:
    """The physics policy selected now (fvb_get_physics)."""
    v = _c_int()
    check(load().fvb_get_physics(ctypes.byref(v)))
    return v.value


class physics:
    """Context manager: run the block's steps with physics policy ``which``
    (FVB_PHYSICS_EULER / FVB_PHYSICS_EULER_PLAIN, fvb_set_physics; plans
    created inside record it).

    with physics(FVB_PHYSICS_EULER_PLAIN): ...
    """

    def __init__(self, which: int) -> None:
        self.which = which

    def __enter__(self):
        lib = load()
        old = _c_int()
        check(lib.fvb_get_physics(ctypes.byref(old)))
        self.old = old.value
        check(lib.fvb_set_physics(self.which))
        return self

    def __exit__(self, *exc):
        check(load().fvb_set_physics(self.old))
