"""CPU oracle for the batched Rusanov FV step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module; the product package
(``paper_2306_16731_b200``) never does, and fails loudly when its CUDA
library is missing instead of falling back here.

Three restatements of the reference algorithm live here, all bit-exact to
``run_sequential`` (pkg/src/patchbench/executors.py:219-270):

* ``step_c`` -- ctypes binding of ``fv_oracle.c`` (literal sequential
  restatement, OpenMP over patches); the fast checker for large batches.
* ``step_numpy`` -- numpy restatement vectorised over all patches of an SoA
  batch, following the vectorised microkernels
  (pkg/src/patchbench/microkernels.py:250-361) term for term.
* ``init_field_soa`` / ``lcg_jump`` -- the seeded field of
  pkg/src/patchbench/bench.py:89-133 with O(log n) jump-ahead.

Parity pin: tests/test_oracle.py compares all of them with fixtures that
``oracle/gen_golden.py`` produced by importing the reference itself, with
SURVEY.md Appendix B's SHA-256 table, and with the reference's frozen LCG
first-cell KAT (pkg/tests/test_bench.py:46-69).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libfv_oracle.so"

LCG_A = 6364136223846793005
LCG_C = 1442695040888963407
MASK64 = (1 << 64) - 1

_lib = None


def build() -> Path:
    """Compile fv_oracle.c with the committed Makefile (no-op when fresh)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.fvo_step_soa.restype = ctypes.c_double
        L.fvo_step_soa.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_int,
        ]
        L.fvo_init_field_soa.restype = None
        L.fvo_init_field_soa.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
        ]
        L.fvo_lcg_jump.restype = ctypes.c_uint64
        L.fvo_lcg_jump.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.fvo_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


# ----------------------------------------------------------------------
# sizes and layouts (pkg/src/patchbench/patchdata.py:61-199)
# ----------------------------------------------------------------------


def sizes(d: int, p: int, t: int) -> tuple[int, int, int]:
    """(N unknowns, haloed cells per patch, interior cells per patch)."""
    return d + 2, (p + 2) ** d, p**d


def soa_to_aos_patches(arr: np.ndarray, d: int, p: int, t: int, haloed: bool) -> np.ndarray:
    """SoA batch (k*T*M + patch*M + lin) -> concatenated per-patch AoS arrays
    ((patch*M + lin)*N + k), i.e. ScatteredPatchSet order (memory.py:60-64)."""
    n = d + 2
    m = (p + 2) if haloed else p
    M = m**d
    return np.ascontiguousarray(arr.reshape(n, t, M).transpose(1, 2, 0)).reshape(-1)


def aos_patches_to_soa(arr: np.ndarray, d: int, p: int, t: int, haloed: bool) -> np.ndarray:
    n = d + 2
    m = (p + 2) if haloed else p
    M = m**d
    return np.ascontiguousarray(arr.reshape(t, M, n).transpose(2, 0, 1)).reshape(-1)


def sha16(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest()[:16]


# ----------------------------------------------------------------------
# LCG field (pkg/src/patchbench/bench.py:89-133)
# ----------------------------------------------------------------------


def lcg_jump(state: int, steps: int) -> int:
    """State after ``steps`` draws of s <- a*s + c mod 2^64."""
    acc_a, acc_c, a, c = 1, 0, LCG_A, LCG_C
    while steps:
        if steps & 1:
            acc_a = (acc_a * a) & MASK64
            acc_c = (acc_c * a + c) & MASK64
        c = ((a + 1) * c) & MASK64
        a = (a * a) & MASK64
        steps >>= 1
    return (acc_a * state + acc_c) & MASK64


def init_field_soa(d: int, p: int, t: int, seed: int, gamma: float = 1.4,
                   threads: int = 0) -> np.ndarray:
    """Haloed SoA input batch holding the reference's ``init_field`` bits."""
    n, M, _ = sizes(d, p, t)
    q = np.empty(n * t * M, dtype=np.float64)
    lib().fvo_init_field_soa(d, p, t, seed & MASK64, gamma, q.ctypes.data, 0, t, threads)
    return q


def init_field_python(d: int, p: int, t: int, seed: int, gamma: float = 1.4) -> np.ndarray:
    """Pure-Python restatement of init_field (small cases; pins the C one)."""
    n, M, _ = sizes(d, p, t)
    q = np.empty((n, t, M), dtype=np.float64)
    state = seed & MASK64

    def uni(lo, hi):
        nonlocal state
        state = (state * LCG_A + LCG_C) & MASK64
        return lo + (hi - lo) * ((state >> 11) * 2.0**-53)

    for patch in range(t):
        for lin in range(M):
            rho = uni(0.5, 2.0)
            u = [uni(-0.5, 0.5) for _ in range(d)]
            pr = uni(0.5, 2.0)
            ke = u[0] * u[0] + u[1] * u[1]
            if d == 3:
                ke = ke + u[2] * u[2]
            q[0, patch, lin] = rho
            for i in range(d):
                q[1 + i, patch, lin] = rho * u[i]
            q[d + 1, patch, lin] = pr / (gamma - 1.0) + 0.5 * rho * ke
    return q.reshape(-1)


# ----------------------------------------------------------------------
# the step
# ----------------------------------------------------------------------


def step_c(d: int, p: int, t: int, q_in: np.ndarray, dt: float = 1e-3, h: float = 0.1,
           gamma: float = 1.4, with_reduction: bool = True, threads: int = 0,
           lam_patch: bool = False):
    """Returns (q_out SoA, reduced or None[, per-patch maxima])."""
    n, M, Mi = sizes(d, p, t)
    q_in = np.ascontiguousarray(q_in, dtype=np.float64)
    assert q_in.size == n * t * M
    out = np.zeros(n * t * Mi, dtype=np.float64)
    lp = np.zeros(t, dtype=np.float64) if lam_patch else None
    red = lib().fvo_step_soa(d, p, t, q_in.ctypes.data, out.ctypes.data, dt, h, gamma,
                             int(with_reduction), lp.ctypes.data if lp is not None else None,
                             threads)
    red = red if with_reduction else None
    return (out, red, lp) if lam_patch else (out, red)


def _pressure(q, d, gamma):
    ke = q[1] * q[1] + q[2] * q[2]
    if d == 3:
        ke = ke + q[3] * q[3]
    return (gamma - 1.0) * (q[d + 1] - ke / (2.0 * q[0]))


def step_numpy(d: int, p: int, t: int, q_in: np.ndarray, dt: float = 1e-3, h: float = 0.1,
               gamma: float = 1.4, with_reduction: bool = True):
    """Vectorised restatement over the whole SoA batch (microkernels.py:265-361).

    Arrays are viewed as [k, patch, c_{d-1}, ..., c_0] so axis ``a`` of the
    reference is numpy axis ``-1-a``.
    """
    n, M, Mi = sizes(d, p, t)
    m = p + 2
    q = np.asarray(q_in, dtype=np.float64).reshape((n, t) + (m,) * d)
    inner = (slice(None), slice(None)) + (slice(1, m - 1),) * d
    out = q[inner].copy()
    scale = dt / h
    for a in range(d):
        ax = 2 + (d - 1 - a)  # numpy axis of reference axis a

        def sl(lo, hi):
            s = [slice(None), slice(None)] + [slice(1, m - 1)] * d
            s[ax] = slice(lo, hi)
            return tuple(s)

        # flux / eigenvalue over c_a in [-1, p] (all of the axis), others interior
        qa = q[sl(0, m)]
        pr = _pressure(qa, d, gamma)
        rho = qa[0]
        energy = qa[d + 1]
        un = qa[1 + a] / rho
        f = np.empty_like(qa)
        f[0] = qa[1 + a]
        for i in range(d):
            f[1 + i] = qa[1 + i] * un + pr if i == a else qa[1 + i] * un
        f[d + 1] = un * (energy + pr)
        lam = np.abs(qa[1 + a] / rho) + np.sqrt(gamma * pr / rho)

        def shift(x, lo, hi, has_k=True):
            s = [slice(None)] * x.ndim
            s[ax if has_k else ax - 1] = slice(lo, hi)
            return x[tuple(s)]

        f_l, f_v, f_r = shift(f, 0, m - 2), shift(f, 1, m - 1), shift(f, 2, m)
        q_l, q_v, q_r = shift(qa, 0, m - 2), shift(qa, 1, m - 1), shift(qa, 2, m)
        lam_l, lam_v, lam_r = (shift(lam, 0, m - 2, False), shift(lam, 1, m - 1, False),
                               shift(lam, 2, m, False))
        w_l = np.maximum(lam_l, lam_v)
        w_r = np.maximum(lam_v, lam_r)
        f_face_l = 0.5 * (f_l + f_v) - 0.5 * w_l * (q_v - q_l)
        f_face_r = 0.5 * (f_v + f_r) - 0.5 * w_r * (q_r - q_v)
        out = out + scale * (f_face_l - f_face_r)
    reduced = None
    if with_reduction:
        pr = _pressure(out, d, gamma)
        rho = out[0]
        c = np.sqrt(gamma * pr / rho)
        value = np.abs(out[1] / rho) + c
        for a in range(1, d):
            value = np.maximum(value, np.abs(out[1 + a] / rho) + c)
        reduced = max(0.0, float(value.max()))
    return np.ascontiguousarray(out).reshape(-1), reduced


def default_threads() -> int:
    """All host cores this process may run on -- not OMP_NUM_THREADS, which
    torchrun pins to 1 per rank (the CPU baseline must use the whole host)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        cores = os.cpu_count() or 1
    return max(1, cores)


if os.environ.get("FVB_ORACLE_AUTOBUILD", "1") == "1" and not LIB_PATH.exists():
    try:
        build()
    except Exception:  # pragma: no cover - surfaced when lib() is used
        pass


def refresh_halos_soa(d: int, p: int, grid, interior: np.ndarray) -> np.ndarray:
    """Haloed SoA input rebuilt from the interior SoA output on a periodic
    patch grid (patch index ix + px*(iy + py*iz)); the checker for
    fvb_refresh_halos.  Builds the periodic global field, pads it by one
    cell, and cuts every patch's haloed window."""
    n = d + 2
    grid = tuple(int(g) for g in grid)
    t = int(np.prod(grid))
    blocks = np.asarray(interior).reshape((n,) + tuple(reversed(grid)) + (p,) * d)
    # [k, iz, iy, ix, cz, cy, cx] -> global [k, z, y, x]
    if d == 2:
        field = blocks.transpose(0, 1, 3, 2, 4).reshape(n, grid[1] * p, grid[0] * p)
    else:
        field = blocks.transpose(0, 1, 4, 2, 5, 3, 6).reshape(n, grid[2] * p, grid[1] * p,
                                                            grid[0] * p)
    padded = np.pad(field, [(0, 0)] + [(1, 1)] * d, mode="wrap")
    m = p + 2
    out = np.empty((n, t) + (m,) * d)
    for patch in range(t):
        ix = patch % grid[0]
        iy = (patch // grid[0]) % grid[1]
        if d == 2:
            out[:, patch] = padded[:, iy * p:iy * p + m, ix * p:ix * p + m]
        else:
            iz = patch // (grid[0] * grid[1])
            out[:, patch] = padded[:, iz * p:iz * p + m, iy * p:iy * p + m, ix * p:ix * p + m]
    return out.reshape(-1)
