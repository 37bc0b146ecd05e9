"""Batch shapes, layouts and device field views.

Mirrors the parts of pkg/src/patchbench/patchdata.py the hot path needs:
``BatchShape`` (:61-102), ``Layout`` (:49-58) and the enumerators
``cell_linear`` / ``linear_offset`` (:122-168), plus ``DeviceFieldView`` --
the GPU analogue of ``FlatFieldView`` (:293-315): one contiguous float64
CUDA tensor holding a field in the device layout, SoA over cells
(``k*T*M + patch*M + lin``).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

__all__ = ["Layout", "LAYOUT_CODES", "BatchShape", "cell_linear", "linear_offset", "DeviceFieldView",
           "relayout"]


class Layout(Enum):
    AOS = "aos"      # unknown fastest within a volume
    SOA = "soa"      # unknown slowest across the batch (the default device layout)
    AOSOA = "aosoa"  # per-patch SoA blocks


# the reference's _LAYOUT_CODES (patchdata.py:57) = include/fvb.h FVB_LAYOUT_*
LAYOUT_CODES = {Layout.AOS: 0, Layout.SOA: 1, Layout.AOSOA: 2}


@dataclass(frozen=True)
class BatchShape:
    """d, volumes per axis p, patch count T (patchdata.py:61-102)."""

    dim: int
    patch_size: int
    patch_count: int

    def __post_init__(self) -> None:
        if self.dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {self.dim}")
        if self.patch_size < 2:
            raise ValueError(f"patch_size must be >= 2, got {self.patch_size}")
        if self.patch_count < 1:
            raise ValueError(f"patch_count must be >= 1, got {self.patch_count}")

    unknowns = property(lambda self: self.dim + 2)
    haloed_extent = property(lambda self: self.patch_size + 2)
    haloed_cells = property(lambda self: self.haloed_extent ** self.dim)
    interior_cells = property(lambda self: self.patch_size ** self.dim)
    input_size = property(lambda self: self.unknowns * self.haloed_cells * self.patch_count)
    output_size = property(lambda self: self.unknowns * self.interior_cells * self.patch_count)

    def extent(self, haloed: bool) -> int:
        return self.haloed_extent if haloed else self.patch_size

    def with_patches(self, patch_count: int) -> "BatchShape":
        return BatchShape(self.dim, self.patch_size, patch_count)


def cell_linear(shape: BatchShape, haloed: bool, cell: Sequence[int]) -> int:
    """Coordinate 0 fastest; haloed coordinates start at -1 (patchdata.py:122-129)."""
    m, shift, lin = shape.extent(haloed), (1 if haloed else 0), 0
    for c in reversed(cell):
        lin = lin * m + c + shift
    return lin


def linear_offset(layout: Layout, shape: BatchShape, haloed: bool, patch: int,
                  cell: Sequence[int], unknown: int) -> int:
    """Storage offset of (patch, cell, unknown) (patchdata.py:142-168)."""
    md = shape.extent(haloed) ** shape.dim
    lin = cell_linear(shape, haloed, cell)
    n = shape.unknowns
    if layout is Layout.AOS:
        return (patch * md + lin) * n + unknown
    if layout is Layout.SOA:
        return unknown * shape.patch_count * md + patch * md + lin
    return patch * n * md + unknown * md + lin


class DeviceFieldView:
    """A batch field resident in HBM: contiguous float64 CUDA tensor in one
    of the reference's layouts (SoA by default).

    ``haloed`` selects the input ((p+2)^d cells per patch) or output (p^d)
    extent.  Replaces FlatFieldView on the GPU path; the kernels address it
    by pointer arithmetic (include/fvb.h "Batch layout", fvb_layout).
    """

    def __init__(self, tensor, shape: BatchShape, haloed: bool, layout: Layout = Layout.SOA) -> None:
        import torch

        if tensor.dtype != torch.float64 or not tensor.is_cuda or not tensor.is_contiguous():
            raise ValueError("DeviceFieldView needs a contiguous float64 CUDA tensor")
        expected = shape.unknowns * shape.extent(haloed) ** shape.dim * shape.patch_count
        if tensor.numel() != expected:
            raise ValueError(f"tensor has {tensor.numel()} entries, expected {expected}")
        self.tensor = tensor
        self.shape = shape
        self.haloed = haloed
        if not isinstance(layout, Layout):
            raise TypeError(f"layout must be a Layout, got {layout!r}")
        self.layout = layout

    @property
    def unknowns(self) -> int:
        return self.shape.unknowns

    def data_ptr(self) -> int:
        return self.tensor.data_ptr()

    def as_array(self):
        """[unknown, patch, lin] view of the tensor (SoA views only)."""
        if self.layout is not Layout.SOA:
            raise ValueError("as_array() is the SoA view; relayout() first")
        return self.tensor.view(self.shape.unknowns, self.shape.patch_count, -1)


def relayout(view: DeviceFieldView, layout: Layout, out=None) -> DeviceFieldView:
    """The same field in another layout (one permutation kernel, fvb_relayout)."""
    import torch

    from . import _lib

    if out is None:
        out = torch.empty_like(view.tensor)
    elif (out.dtype != torch.float64 or out.device != view.tensor.device or not out.is_contiguous()
          or out.numel() != view.tensor.numel()):
        raise ValueError("out must be a contiguous float64 tensor like the view's, on its device")
    s = view.shape
    with torch.cuda.device(out.device):  # the library launches on the current device
        _lib.check(_lib.load().fvb_relayout(s.dim, s.patch_size, s.patch_count, int(view.haloed),
                                            LAYOUT_CODES[view.layout], LAYOUT_CODES[layout],
                                            view.data_ptr(), out.data_ptr(),
                                            torch.cuda.current_stream(out.device).cuda_stream))
    return DeviceFieldView(out, s, view.haloed, layout)
