"""Host twin of the user microkernels (pkg/src/patchbench/equations.py).

The device kernels call the CUDA twins in csrc/euler.cuh; this module keeps
the reference's Python signatures for the user-function interface
(``flux(q, axis, params, check)``, ``max_eigenvalue(q, axis, params, check)``)
so code written against the reference keeps importing them, and so the
tests can compare the device twins with the host ones state by state.
Same closure, same association of every operation.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

from .errors import InvalidStateError

__all__ = ["DEFAULT_GAMMA", "EulerParameters", "InvalidStateError", "pressure", "flux",
           "max_eigenvalue", "is_admissible"]

DEFAULT_GAMMA = 1.4


@dataclass(frozen=True)
class EulerParameters:
    """Ideal-gas closure: adiabatic exponent gamma > 1."""

    gamma: float = DEFAULT_GAMMA

    def __post_init__(self) -> None:
        if not self.gamma > 1.0:
            raise ValueError(f"adiabatic exponent must exceed 1, got {self.gamma}")


def _dim(q: Sequence[float]) -> int:
    if len(q) not in (4, 5):
        raise ValueError(f"state has {len(q)} entries; expected d+2 with d in {{2,3}}")
    return len(q) - 2


def pressure(q: Sequence[float], params: EulerParameters, check: bool = False) -> float:
    d = _dim(q)
    rho = q[0]
    if check and not rho > 0.0:
        raise InvalidStateError(f"non-positive density {rho}")
    kinetic = q[1] * q[1] + q[2] * q[2]
    if d == 3:
        kinetic = kinetic + q[3] * q[3]
    pr = (params.gamma - 1.0) * (q[d + 1] - kinetic / (2.0 * rho))
    if check and not pr > 0.0:
        raise InvalidStateError(f"non-positive pressure {pr} for state {tuple(q)}")
    return pr


def _axis_ok(d: int, axis: int) -> None:
    if not 0 <= axis < d:
        raise ValueError(f"axis {axis} out of range for d={d}")


def flux(q: Sequence[float], axis: int, params: EulerParameters,
         check: bool = False) -> tuple[float, ...]:
    d = _dim(q)
    _axis_ok(d, axis)
    pr = pressure(q, params, check)
    vel = q[1 + axis] / q[0]
    mom = [q[1 + i] * vel for i in range(d)]
    mom[axis] = q[1 + axis] * vel + pr
    return (q[1 + axis], *mom, vel * (q[d + 1] + pr))


def max_eigenvalue(q: Sequence[float], axis: int, params: EulerParameters,
                   check: bool = False) -> float:
    d = _dim(q)
    _axis_ok(d, axis)
    pr = pressure(q, params, check)
    return abs(q[1 + axis] / q[0]) + math.sqrt(params.gamma * pr / q[0])


def is_admissible(q: Sequence[float], params: EulerParameters) -> bool:
    try:
        pressure(q, params, check=True)
    except InvalidStateError:
        return False
    return True
