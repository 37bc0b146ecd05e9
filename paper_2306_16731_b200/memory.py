"""Transfer modes between host patches and the device batch (f1 row).

GPU form of pkg/src/patchbench/memory.py.  The host hands over T patches as
per-patch AoS arrays (``ScatteredPatchSet``, :60-96); the device computes on
one SoA batch.  Modes:

* ``EXPLICIT_COPY`` -- fresh device buffers per launch, freed afterwards;
* ``POOLED``        -- device buffers recycled by a ``DeviceArena`` that never
                       frees (allocation counter constant after the first
                       launch, :105-137);
* ``SHARED``        -- the batch already lives in HBM (``DevicePatchSet``):
                       no transfer at all, the USM analogue of computing in
                       place.

Host<->device movement is one DMA of the contiguous pinned AoS block
(``allocate_scattered(pinned=True)`` makes the per-patch arrays views into
it) plus one AoS<->SoA permutation kernel on the device
(``fvb_aos_to_soa`` / ``fvb_soa_to_aos``) -- gather_patches (:240-251) and
scatter_results (:254-265) without a per-patch host loop.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import ShapeMismatchError
from .patchdata import LAYOUT_CODES, BatchShape, DeviceFieldView, Layout

__all__ = ["TransferMode", "ShapeMismatchError", "ScatteredPatchSet", "DevicePatchSet",
           "allocate_scattered", "DeviceArena", "LaunchBuffers", "acquire_buffers",
           "release_buffers", "gather_patches", "scatter_results"]


class TransferMode(Enum):
    SHARED = "shared"
    EXPLICIT_COPY = "copy"
    POOLED = "pooled"


@dataclass
class ScatteredPatchSet:
    """T per-patch AoS arrays: haloed input and interior output (memory.py:60-96).

    ``in_block`` / ``out_block`` (optional) are contiguous backing arrays the
    per-patch arrays are views of -- pinned when made by
    ``allocate_scattered(pinned=True)`` -- which turns gather/scatter into
    single DMAs.
    """

    shape: BatchShape
    inputs: list
    outputs: list
    in_block: np.ndarray | None = None
    out_block: np.ndarray | None = None
    _pinned: list = field(default_factory=list, repr=False)

    def __post_init__(self) -> None:
        s = self.shape
        if len(self.inputs) != s.patch_count or len(self.outputs) != s.patch_count:
            raise ShapeMismatchError("patch array count does not match patch_count")
        nin, nout = s.unknowns * s.haloed_cells, s.unknowns * s.interior_cells
        if any(a.size != nin for a in self.inputs) or any(a.size != nout for a in self.outputs):
            raise ShapeMismatchError("per-patch array size does not match the shape")

    def input_block(self) -> np.ndarray:
        return self.in_block if self.in_block is not None else np.concatenate(self.inputs)

    def output_block_target(self) -> np.ndarray | None:
        return self.out_block

    def clone(self) -> "ScatteredPatchSet":
        c = allocate_scattered(self.shape, pinned=False)
        c.in_block[:] = self.input_block()
        for dst, src in zip(c.outputs, self.outputs):
            dst[:] = src
        return c


def allocate_scattered(shape: BatchShape, pinned: bool = False) -> ScatteredPatchSet:
    """Zeroed patch set whose per-patch arrays view two contiguous blocks."""
    nin, nout = shape.unknowns * shape.haloed_cells, shape.unknowns * shape.interior_cells
    keep = []
    if pinned:
        import torch

        tin = torch.zeros(nin * shape.patch_count, dtype=torch.float64, pin_memory=True)
        tout = torch.zeros(nout * shape.patch_count, dtype=torch.float64, pin_memory=True)
        keep = [tin, tout]
        in_block, out_block = tin.numpy(), tout.numpy()
    else:
        in_block = np.zeros(nin * shape.patch_count)
        out_block = np.zeros(nout * shape.patch_count)
    inputs = [in_block[i * nin:(i + 1) * nin] for i in range(shape.patch_count)]
    outputs = [out_block[i * nout:(i + 1) * nout] for i in range(shape.patch_count)]
    return ScatteredPatchSet(shape, inputs, outputs, in_block, out_block, keep)


@dataclass
class DevicePatchSet:
    """A batch resident in HBM (SoA input + output): SHARED mode's operand."""

    shape: BatchShape
    input: DeviceFieldView
    output: DeviceFieldView

    @classmethod
    def empty(cls, shape: BatchShape, device="cuda", layout: Layout = Layout.SOA) -> "DevicePatchSet":
        import torch

        qi = torch.empty(shape.input_size, dtype=torch.float64, device=device)
        qo = torch.zeros(shape.output_size, dtype=torch.float64, device=device)
        return cls(shape, DeviceFieldView(qi, shape, True, layout),
                   DeviceFieldView(qo, shape, False, layout))


class DeviceArena:
    """Device buffer source with recycling and allocation accounting."""

    def __init__(self, device="cuda") -> None:
        self.device = device
        self.allocation_count = 0
        self.outstanding_bytes = 0
        self.high_water_bytes = 0
        self._pool: dict[tuple, list] = {}

    def allocate(self, count: int):
        import torch

        buf = torch.empty(count, dtype=torch.float64, device=self.device)
        self.allocation_count += 1
        self.outstanding_bytes += count * 8
        self.high_water_bytes = max(self.high_water_bytes, self.outstanding_bytes)
        return buf

    def free(self, buf) -> None:
        self.outstanding_bytes -= buf.numel() * 8

    def acquire(self, key: tuple, count: int):
        stack = self._pool.get(key)
        return stack.pop() if stack else self.allocate(count)

    def recycle(self, key: tuple, buf) -> None:
        self._pool.setdefault(key, []).append(buf)


@dataclass
class LaunchBuffers:
    mode: TransferMode
    shape: BatchShape
    input_view: DeviceFieldView
    output_view: DeviceFieldView
    staging_in: object = None   # device AoS staging (copy / pooled)
    staging_out: object = None
    pooled: list = field(default_factory=list)
    owned: list = field(default_factory=list)


def acquire_buffers(shape: BatchShape, mode: TransferMode, arena: DeviceArena,
                    patches, layout: Layout = Layout.SOA) -> LaunchBuffers:
    if patches.shape != shape:
        raise ShapeMismatchError(f"patch set is {patches.shape}, launch wants {shape}")
    if mode is TransferMode.SHARED:
        if not isinstance(patches, DevicePatchSet):
            raise ValueError("SHARED mode computes in place on a DevicePatchSet "
                             "(device-resident batch); host patches need COPY or POOLED")
        return LaunchBuffers(mode, shape, patches.input, patches.output)
    sizes = [shape.input_size, shape.output_size, shape.input_size, shape.output_size]
    roles = ["input", "output", "stage_in", "stage_out"]
    key = (shape.dim, shape.patch_size, shape.patch_count)
    if mode is TransferMode.EXPLICIT_COPY:
        bufs = [arena.allocate(n) for n in sizes]
        pooled, owned = [], bufs
    else:
        keys = [(r,) + key for r in roles]
        bufs = [arena.acquire(k, n) for k, n in zip(keys, sizes)]
        pooled, owned = list(zip(keys, bufs)), []
    return LaunchBuffers(mode, shape, DeviceFieldView(bufs[0], shape, True, layout),
                         DeviceFieldView(bufs[1], shape, False, layout), bufs[2], bufs[3], pooled,
                         owned)


def release_buffers(buffers: LaunchBuffers, arena: DeviceArena) -> None:
    for key, buf in buffers.pooled:
        arena.recycle(key, buf)
    for buf in buffers.owned:
        arena.free(buf)
    buffers.pooled, buffers.owned = [], []


def _stream():
    import torch

    return torch.cuda.current_stream()


def gather_patches(src: ScatteredPatchSet, buffers: LaunchBuffers) -> None:
    """Host AoS patches -> device input in the batch layout: one H2D DMA
    (straight into the batch for AoS) + one permutation (SoA / AoSoA)."""
    import torch

    s = buffers.shape
    if src.shape != s:
        raise ShapeMismatchError(f"gather from {src.shape} into {s}")
    host = torch.from_numpy(src.input_block())
    layout = buffers.input_view.layout
    if layout is Layout.AOS:
        buffers.input_view.tensor.copy_(host, non_blocking=True)
        return
    buffers.staging_in.copy_(host, non_blocking=True)
    _lib.check(_lib.load().fvb_relayout(s.dim, s.patch_size, s.patch_count, 1, LAYOUT_CODES[Layout.AOS],
                                        LAYOUT_CODES[layout], buffers.staging_in.data_ptr(),
                                        buffers.input_view.data_ptr(), _stream().cuda_stream))


def scatter_results(buffers: LaunchBuffers, dst: ScatteredPatchSet) -> None:
    """Device output in the batch layout -> host AoS patches: one
    permutation (SoA / AoSoA; none for AoS) + one D2H DMA."""
    import torch

    s = buffers.shape
    if dst.shape != s:
        raise ShapeMismatchError(f"scatter from {s} into {dst.shape}")
    layout = buffers.output_view.layout
    src_dev = buffers.output_view.tensor if layout is Layout.AOS else buffers.staging_out
    if layout is not Layout.AOS:
        _lib.check(_lib.load().fvb_relayout(s.dim, s.patch_size, s.patch_count, 0,
                                            LAYOUT_CODES[layout], LAYOUT_CODES[Layout.AOS],
                                            buffers.output_view.data_ptr(),
                                            buffers.staging_out.data_ptr(), _stream().cuda_stream))
    target = dst.output_block_target()
    if target is not None:
        torch.from_numpy(target).copy_(src_dev, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    else:
        host = src_dev.cpu().numpy()
        n = s.unknowns * s.interior_cells
        for i, arr in enumerate(dst.outputs):
            arr[:] = host[i * n:(i + 1) * n]
