"""Multi-GPU sharding of the batched step.

Patches are independent (no cross-patch DAG edges, kernelgraph.py:215-247)
and halos are inputs, so the batch shards by contiguous patch
ranges with no data-path exchange.  The one real exchange is the admissible
time step: every rank needs the global maximum eigenvalue, one 8-byte
``all_reduce(MAX)`` over NCCL (NVLink / NVSwitch) per step.  Max is exact
and order-free, so the reduced eigenvalue -- and dt derived from it -- are
bit-identical for any number of ranks and equal to the 1-GPU / CPU oracle
value.
"""

from __future__ import annotations

from .context import TimeStepContext
from .executors import Realization, step_async
from .kernelgraph import build_plan
from .launch import admissible_dt, init_field_device
from .patchdata import BatchShape, DeviceFieldView

__all__ = ["shard_range", "ShardedStep"]


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) patch range of ``rank``; sizes differ by at most 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def global_max_(lam, group=None):
    """In-place all-reduce(MAX) of a one-element eigenvalue tensor."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(lam, op=dist.ReduceOp.MAX, group=group)
    return lam


class ShardedStep:
    """This rank's shard of a T_total-patch batch, stepped on its GPU.

    ``step()`` enqueues the local kernel(s) and the all-reduce on the current
    stream and returns the global eigenvalue tensor (device); ``dt()`` turns
    it into the admissible time step (host, identical on every rank).
    """

    def __init__(self, dim: int, p: int, total_patches: int, rank: int, world: int,
                 ctx: TimeStepContext, realization: Realization = Realization.PATCH_WISE,
                 seed: int = 0, device="cuda", group=None) -> None:
        import torch

        self.lo, self.hi = shard_range(total_patches, rank, world)
        self.shape = BatchShape(dim, p, self.hi - self.lo)
        self.ctx = ctx
        self.realization = realization
        self.group = group
        self.plan = build_plan(self.shape, True)
        self.inp = init_field_device(self.shape, seed, ctx.params.gamma, device, patch_begin=self.lo)
        self.out = DeviceFieldView(torch.empty(self.shape.output_size, dtype=torch.float64,
                                               device=device), self.shape, False)
        self.lam = torch.zeros(1, dtype=torch.float64, device=device)

    def step(self):
        step_async(self.realization, self.plan, self.inp, self.out, self.ctx, lam=self.lam)
        return global_max_(self.lam, self.group)

    def dt(self, cfl: float = 0.5) -> float:
        return admissible_dt(float(self.lam.item()), self.ctx.h, cfl)
