"""Multi-step driver on a periodic grid of patches.

The reference performs one step and reports the reduced eigenvalue
(SPEC.md:8).  A time-stepping run needs two more things, both added here:
the admissible time step from the eigenvalue (``dt = cfl*h/lambda``,
``fvb_admissible_dt``) and a halo refresh that rebuilds the haloed input of
the next step from the interior output of the last one
(``fvb_refresh_halos``: patches on a periodic px x py (x pz) grid).  Each
step is: fused step (with the current dt) -> eigenvalue -> [all-reduce max]
-> dt for the next step -> halo refresh.  The per-patch eigenvalues
(local-time-stepping input) are available via
``lam_patch``.

``step()`` keeps dt on the host (one eigenvalue read per step).
``step_device()`` keeps it in HBM: the kernels read dt (fvb_step_dt), the
next dt is formed by ``fvb_admissible_dt_dev`` and the simulated time is
accumulated on the device -- no host synchronisation, so ``capture(k)``
records k steps as one CUDA graph and ``replay()`` relaunches them with a
single call.  Both forms give identical bits.
"""

from __future__ import annotations

from . import _lib
from .context import TimeStepContext
from .equations import EulerParameters
from .executors import Realization, step_async
from .kernelgraph import build_plan
from .launch import admissible_dt, init_field_device
from .patchdata import BatchShape, DeviceFieldView

__all__ = ["PatchGridSimulation"]


class PatchGridSimulation:
    def __init__(self, dim: int, p: int, grid: tuple[int, ...], h: float = 0.1,
                 gamma: float = 1.4, cfl: float = 0.5, dt0: float = 1e-3, seed: int = 0,
                 realization: Realization = Realization.PATCH_WISE, device="cuda",
                 per_patch_lambda: bool = False) -> None:
        import torch

        if len(grid) != dim:
            raise ValueError(f"grid {grid} must have {dim} entries")
        self.grid = tuple(int(g) for g in grid) + (1,) * (3 - dim)
        t = 1
        for g in grid:
            t *= int(g)
        self.shape = BatchShape(dim, p, t)
        self.h, self.gamma, self.cfl, self.dt = h, gamma, cfl, dt0
        self.realization = realization
        self.plan = build_plan(self.shape, True)
        self.inp = init_field_device(self.shape, seed, gamma, device)
        self.out = DeviceFieldView(torch.empty(self.shape.output_size, dtype=torch.float64,
                                               device=device), self.shape, False)
        self.lam = torch.zeros(1, dtype=torch.float64, device=device)
        self.lam_patch = (torch.zeros(t, dtype=torch.float64, device=device)
                          if per_patch_lambda else None)
        self.time = 0.0
        self.steps = 0
        self.dt_dev = torch.full((1,), float(dt0), dtype=torch.float64, device=device)
        self.time_dev = torch.zeros(1, dtype=torch.float64, device=device)
        self.graph = None
        self.graph_steps = 0

    def refresh_halos(self) -> None:
        import torch

        s = self.shape
        _lib.check(_lib.load().fvb_refresh_halos(
            s.dim, s.patch_size, self.grid[0], self.grid[1], self.grid[2], self.out.data_ptr(),
            self.inp.data_ptr(), torch.cuda.current_stream().cuda_stream))

    def step(self, group=None) -> float:
        """Advance one step with the current dt; returns the new dt."""
        from .distributed import global_max_

        ctx = TimeStepContext(self.dt, self.h, EulerParameters(self.gamma))
        step_async(self.realization, self.plan, self.inp, self.out, ctx, lam=self.lam,
                   lam_patch=self.lam_patch)
        global_max_(self.lam, group)
        self.refresh_halos()
        self.time += self.dt
        self.steps += 1
        self.dt = admissible_dt(float(self.lam.item()), self.h, self.cfl)
        return self.dt

    def run(self, nsteps: int) -> list[float]:
        return [self.step() for _ in range(nsteps)]

    # ---- device-resident dt: no host sync, CUDA-graph capturable ----------
    def step_device(self, group=None) -> None:
        """Enqueue one step that reads and writes dt in HBM."""
        import torch

        from .distributed import global_max_

        ctx = TimeStepContext(1.0, self.h, EulerParameters(self.gamma))  # dt: self.dt_dev
        step_async(self.realization, self.plan, self.inp, self.out, ctx, lam=self.lam,
                   lam_patch=self.lam_patch, dt_dev=self.dt_dev)
        global_max_(self.lam, group)
        self.time_dev.add_(self.dt_dev)
        _lib.check(_lib.load().fvb_admissible_dt_dev(
            self.lam.data_ptr(), self.h, self.cfl, self.dt_dev.data_ptr(),
            torch.cuda.current_stream().cuda_stream))
        self.refresh_halos()

    def run_device(self, nsteps: int) -> None:
        for _ in range(nsteps):
            self.step_device()
        self.steps += nsteps

    def capture(self, nsteps: int) -> None:
        """Record ``nsteps`` device-dt steps as one CUDA graph."""
        import torch

        self.step_device()  # warm: library plans / first-launch setup outside the capture
        torch.cuda.synchronize()
        self.steps += 1
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            for _ in range(nsteps):
                self.step_device()
        self.graph_steps = nsteps

    def replay(self) -> None:
        self.graph.replay()
        self.steps += self.graph_steps

    def sync_host(self) -> tuple[float, float]:
        """(current dt, simulated time) read back from the device."""
        self.dt = float(self.dt_dev.item())
        self.time = float(self.time_dev.item())
        return self.dt, self.time
