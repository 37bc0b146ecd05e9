"""Launch metadata (pkg/src/patchbench/microkernels.py:54-67)."""

from __future__ import annotations

from dataclasses import dataclass

from .equations import EulerParameters

__all__ = ["TimeStepContext"]


@dataclass(frozen=True)
class TimeStepContext:
    """dt, volume edge length h, closure parameters, admissibility checks."""

    dt: float
    h: float
    params: EulerParameters
    check: bool = False

    def __post_init__(self) -> None:
        if not self.dt > 0.0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if not self.h > 0.0:
            raise ValueError(f"h must be positive, got {self.h}")

    @property
    def scale(self) -> float:
        """dt/h as the kernels use it (one IEEE division, microkernels.py:179)."""
        return self.dt / self.h
