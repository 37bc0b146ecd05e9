"""Transfer modes between host patches and the device (f1 row).

GPU form of pkg/src/patchbench/memory.py.  The host hands over T patches as
independently allocated per-patch AoS arrays (``ScatteredPatchSet``,
:60-96); the GPU reaches them through pointer tables:

* ``SHARED``        -- compute in place on the per-patch arrays: the step
                       kernels read the haloed inputs and write the interior
                       outputs through device tables of their (host-mapped)
                       addresses -- no batch buffers, no copies (the USM
                       analogue, :162-228; ScatteredFieldView,
                       patchdata.py:318-334);
* ``EXPLICIT_COPY`` -- gather into freshly allocated device batch buffers in
                       the requested layout, step, scatter back, free;
* ``POOLED``        -- the same with buffers recycled by a ``DeviceArena``
                       that never frees (allocation counter constant after
                       the first launch, :105-137).

COPY / POOLED launches over arrays that are not pinned are host-staged (the
library gathers chunks into pinned memory and DMAs them, no registration).
The GPU addresses host memory directly (SHARED, check mode) when it is
pinned or registered: ``allocate_scattered(pinned=True)`` / ``init_field``
make pinned sets; any other set is registered for the duration of each launch
(``ScatteredPatchSet.addressable``: the page-merged spans of its arrays,
refcounted in libfvb, unregistered after the launch synchronised).  The
registration is transient on purpose: it covers whole pages, and a pageable
cudaMemcpy of ANY other buffer that starts inside a registered page and runs
past it fails with cudaErrorInvalidValue (measured on B200, driver 580) --
heap arrays registered for good would break unrelated ``tensor.cpu()``
copies.  ``ScatteredPatchSet.pin`` keeps the registration for the set's
lifetime, for callers whose arrays own their pages.  gather / scatter are the table
kernels of csrc/xfer.cu (zero-copy PCIe reads / writes, permuted into the
batch layout on the way); run_launch pipelines them with the step over
patch chunks (fvb_launch_table).  Per-patch pointers come from the
``_hostptr`` extension (one C loop, cached while the patch lists are
unchanged) -- no per-patch Python loop and no ``np.concatenate``.
"""

from __future__ import annotations

import contextlib
import ctypes
import struct
import weakref
from pathlib import Path
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import ShapeMismatchError
from .patchdata import LAYOUT_CODES, BatchShape, DeviceFieldView, Layout

__all__ = ["TransferMode", "ShapeMismatchError", "ScatteredPatchSet", "DevicePatchSet", "PatchList",
           "HostPatchView", "DeviceBatch", "GpuScratchArrays", "allocate_scattered", "DeviceArena",
           "LaunchBuffers", "acquire_buffers", "release_buffers", "gather_patches",
           "scatter_results", "pinned_scattered", "dump_batch", "load_batch", "read_batch_file",
           "write_batch_file"]


class TransferMode(Enum):
    SHARED = "shared"
    EXPLICIT_COPY = "copy"
    POOLED = "pooled"


def _hostptr():
    try:
        from . import _hostptr as mod
    except ImportError:  # built with the library (build.py)
        from . import build as _build

        _build.build_hostptr()
        from . import _hostptr as mod
    return mod


class PatchList(list):
    """A list of per-patch arrays that counts its mutations, so the cached
    pointer table of a ScatteredPatchSet stays valid until one happens."""

    version = 0

    def _bump(self):
        self.version += 1

    def __setitem__(self, i, v):
        self._bump()
        super().__setitem__(i, v)

    def __delitem__(self, i):
        self._bump()
        super().__delitem__(i)

    def __iadd__(self, other):
        self._bump()
        return super().__iadd__(other)

    def __imul__(self, n):
        self._bump()
        return super().__imul__(n)

    def append(self, v):
        self._bump()
        super().append(v)

    def extend(self, v):
        self._bump()
        super().extend(v)

    def insert(self, i, v):
        self._bump()
        super().insert(i, v)

    def pop(self, *a):
        self._bump()
        return super().pop(*a)

    def remove(self, v):
        self._bump()
        super().remove(v)

    def clear(self):
        self._bump()
        super().clear()

    def sort(self, *a, **k):
        self._bump()
        super().sort(*a, **k)

    def reverse(self):
        self._bump()
        super().reverse()


class _PinHandle:
    """A libfvb fvb_pin handle; released (unregistering what no other
    handle holds) when its owner is collected -- the arrays stay referenced
    until then, so a registration never outlives the memory."""

    def __init__(self, handle: ctypes.c_void_p, keep) -> None:
        self._fin = weakref.finalize(self, _unpin, handle.value, keep)

    def release(self) -> None:
        self._fin()


def _unpin(handle, keep) -> None:  # keep: the arrays / blocks, alive until here
    if handle:
        try:
            _lib.load().fvb_host_unpin(ctypes.c_void_p(handle))
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


@dataclass
class ScatteredPatchSet:
    """T per-patch AoS arrays: haloed input and interior output (memory.py:60-96).

    The arrays may be independently allocated anywhere (the reference's
    ``allocate_scattered``) or views into pinned blocks
    (``allocate_scattered(pinned=True)``, ``init_field``).  ``in_block`` /
    ``out_block`` are those blocks when they exist.
    """

    shape: BatchShape
    inputs: list
    outputs: list
    in_block: np.ndarray | None = None
    out_block: np.ndarray | None = None
    _keep: list = field(default_factory=list, repr=False)
    _sized: bool = field(default=False, repr=False)  # arrays made here: sizes known

    def __post_init__(self) -> None:
        s = self.shape
        if len(self.inputs) != s.patch_count or len(self.outputs) != s.patch_count:
            raise ShapeMismatchError("patch array count does not match patch_count")
        if not isinstance(self.inputs, PatchList):
            self.inputs = PatchList(self.inputs)
        if not isinstance(self.outputs, PatchList):
            self.outputs = PatchList(self.outputs)
        self._tables = {}
        self._pin = None
        if self._sized:
            return
        nin, nout = s.unknowns * s.haloed_cells, s.unknowns * s.interior_cells
        for i, a in enumerate(self.inputs):
            if np.size(a) != nin:
                raise ShapeMismatchError(f"input patch {i} has {np.size(a)} != {nin} entries")
        for i, a in enumerate(self.outputs):
            if np.size(a) != nout:
                raise ShapeMismatchError(f"output patch {i} has {np.size(a)} != {nout} entries")

    # ---- pointer tables ---------------------------------------------------
    def _table(self, which: str) -> np.ndarray:
        lst = self.inputs if which == "in" else self.outputs
        if not isinstance(lst, PatchList):  # reassigned attribute
            lst = PatchList(lst)
            setattr(self, "inputs" if which == "in" else "outputs", lst)
        key = (id(lst), lst.version, len(lst))
        hit = self._tables.get(which)
        if hit is not None and hit[0] == key:
            return hit[1]
        s = self.shape
        count = s.unknowns * (s.haloed_cells if which == "in" else s.interior_cells)
        if len(lst) != s.patch_count:
            raise ShapeMismatchError("patch array count does not match patch_count")
        tab = np.empty(len(lst), dtype=np.uint64)
        try:
            _hostptr().pointer_table(lst, count, tab, which == "out")
        except ValueError as exc:
            raise ShapeMismatchError(str(exc)) from None
        self._tables[which] = (key, tab)
        return tab

    def input_table(self) -> np.ndarray:
        """uint64 addresses of the T input arrays (cached)."""
        return self._table("in")

    def output_table(self) -> np.ndarray:
        """uint64 addresses of the T output arrays (cached)."""
        return self._table("out")

    # ---- device addressability ---------------------------------------------
    def _first_unpinned(self) -> int:
        lib = _lib.load()
        s = self.shape
        bad = ctypes.c_int64()
        for tab, n in ((self.input_table(), s.unknowns * s.haloed_cells),
                       (self.output_table(), s.unknowns * s.interior_cells)):
            _lib.check(lib.fvb_host_accessible(tab.ctypes.data, len(tab), n * 8, ctypes.byref(bad)))
            if bad.value >= 0:
                return bad.value
        return -1

    def is_device_accessible(self) -> bool:
        return self._first_unpinned() < 0

    def _register(self) -> list:
        lib = _lib.load()
        s = self.shape
        handles = []
        for tab, n in ((self.input_table(), s.unknowns * s.haloed_cells),
                       (self.output_table(), s.unknowns * s.interior_cells)):
            h = ctypes.c_void_p()
            _lib.check(lib.fvb_host_pin(tab.ctypes.data, len(tab), n * 8, ctypes.byref(h)))
            handles.append(_PinHandle(h, (list(self.inputs), list(self.outputs))))
        return handles

    def pin(self) -> None:
        """Register every array for the set's lifetime (persistent).  Only
        safe when the arrays own their pages: a pageable cudaMemcpy of another
        buffer starting inside a registered page fails (see the module
        docstring).  Launches register unpinned sets transiently instead."""
        if self.is_device_accessible():
            return
        self._pin = self._register()

    def unpin(self) -> None:
        for h in self._pin or []:
            h.release()
        self._pin = None

    @contextlib.contextmanager
    def addressable(self, sync=None):
        """Device-addressable inside the block: pinned blocks and pinned sets
        as they are, anything else registered now and unregistered on exit --
        after ``sync()`` (the caller's stream / device synchronisation: no
        kernel may still address the pages)."""
        if self.is_device_accessible():
            yield self
            return
        handles = self._register()
        try:
            yield self
        finally:
            try:
                if sync is not None:
                    sync()
            finally:
                for h in handles:
                    h.release()

    # ---- reference API -------------------------------------------------------
    def input_view(self) -> "HostPatchView":
        return HostPatchView(self, True)

    def output_view(self) -> "HostPatchView":
        return HostPatchView(self, False)

    def input_block(self) -> np.ndarray:
        """The inputs as one contiguous AoS array (a copy unless blocked)."""
        return self.in_block if self.in_block is not None else np.concatenate(self.inputs)

    def clone(self) -> "ScatteredPatchSet":
        """Deep copy (memory.py:90-96).  A pinned blocked set clones into a
        new pinned blocked set, any other set into independent arrays."""
        if self.in_block is not None and self._keep:
            c = allocate_scattered(self.shape, pinned=True, zero=False)
            c.in_block[:] = self.in_block
            c.out_block[:] = self.out_block
            return c
        return ScatteredPatchSet(self.shape, [np.array(a, dtype=np.float64, copy=True) for a in self.inputs],
                                 [np.array(a, dtype=np.float64, copy=True) for a in self.outputs])


def allocate_scattered(shape: BatchShape, pinned: bool = False, zero: bool = True) -> ScatteredPatchSet:
    """Zeroed patch set.  pinned=False: T independently allocated arrays per
    direction (the reference's allocate_scattered, memory.py:99-104).
    pinned=True: views into two pinned host blocks, device-addressable
    (zero=False leaves them uninitialised, for callers that fill them)."""
    nin, nout = shape.unknowns * shape.haloed_cells, shape.unknowns * shape.interior_cells
    t = shape.patch_count
    if not pinned:
        return ScatteredPatchSet(shape, [np.zeros(nin) for _ in range(t)],
                                 [np.zeros(nout) for _ in range(t)], _sized=True)
    import torch

    make = torch.zeros if zero else torch.empty
    tin = make(nin * t, dtype=torch.float64, pin_memory=True)
    tout = make(nout * t, dtype=torch.float64, pin_memory=True)
    in_block, out_block = tin.numpy(), tout.numpy()
    inputs = [in_block[i * nin:(i + 1) * nin] for i in range(t)]
    outputs = [out_block[i * nout:(i + 1) * nout] for i in range(t)]
    sc = ScatteredPatchSet(shape, inputs, outputs, in_block, out_block, [tin, tout], _sized=True)
    lib = _lib.load()
    handles = []
    for blk in (tin, tout):
        h = ctypes.c_void_p()
        _lib.check(lib.fvb_host_note_pinned(blk.data_ptr(), blk.numel() * 8, ctypes.byref(h)))
        handles.append(_PinHandle(h, blk))
    sc._keep.append(handles)
    return sc


def pinned_scattered(shape: BatchShape) -> ScatteredPatchSet:
    return allocate_scattered(shape, pinned=True)


class HostPatchView:
    """The per-patch arrays of a ScatteredPatchSet as a field view
    (ScatteredFieldView, patchdata.py:318-334): what SHARED mode computes on."""

    def __init__(self, patches: ScatteredPatchSet, haloed: bool) -> None:
        self.patches = patches
        self.shape = patches.shape
        self.haloed = haloed
        self.layout = Layout.AOS

    @property
    def unknowns(self) -> int:
        return self.shape.unknowns

    def table(self) -> np.ndarray:
        return self.patches.input_table() if self.haloed else self.patches.output_table()

    def device_table(self, device=None):
        """The pointer table as a CUDA uint64 tensor.  The arrays must be
        device-addressable (inside ``ScatteredPatchSet.addressable()``, or
        pinned)."""
        import torch

        bad = self.patches._first_unpinned()
        if bad >= 0:
            raise ValueError(f"patch {bad} is not in device-addressable host memory: use the set "
                             "inside ScatteredPatchSet.addressable() or pin() it")
        # via a pinned copy: the table is pageable and may share a page with
        # registered patch arrays, where a pageable copy fails (module docstring)
        tab = self.table().view(np.int64)
        staged = torch.empty(len(tab), dtype=torch.int64, pin_memory=True)
        staged.numpy()[:] = tab
        return staged.to(device or "cuda")


@dataclass
class DevicePatchSet:
    """A batch resident in HBM (input + output in one layout)."""

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


@dataclass
class DeviceBatch:
    """The device batch of one COPY / POOLED launch (PatchBatch, patchdata.py:231-248)."""

    shape: BatchShape
    layout: Layout
    input: DeviceFieldView
    output: DeviceFieldView


class _LazyBuffer:
    """An arena buffer whose device memory is allocated on first use (the
    fused flavour never touches the step temporaries)."""

    def __init__(self, count: int, device) -> None:
        self.count = count
        self.device = device
        self._t = None
        self.plans: dict = {}  # libfvb plans bound to this buffer set (GpuScratchArrays.plan)

    def numel(self) -> int:
        return self.count

    @property
    def tensor(self):
        if self._t is None:
            import torch

            self._t = torch.empty(self.count, dtype=torch.float64, device=self.device)
        return self._t


class GpuScratchArrays:
    """Per-axis flux / wave-speed temporaries of the cascade and graph
    flavours (ScratchArrays, microkernels.py:70-112; tight to the flux
    range), owned by the arena.  ``plan(flavour)`` binds a libfvb plan to
    them (cached: a pooled arena's graph is instantiated once)."""

    def __init__(self, shape: BatchShape, flux: list, lam: list) -> None:
        self.shape = shape
        self.flux = flux
        self.lam = lam
        self._plans: dict = {}

    @staticmethod
    def sizes(shape: BatchShape) -> tuple[int, int]:
        f, l_ = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().fvb_scratch_doubles(shape.dim, shape.patch_size, shape.patch_count,
                                                   ctypes.byref(f), ctypes.byref(l_)))
        return f.value, l_.value

    def plan(self, flavour: int):
        # cached on the first temporary: a pooled arena hands the same
        # buffers to every launch, so its graph is instantiated once; a plan
        # records the physics policy selected when it is made (fvb_set_physics)
        cache = getattr(self.flux[0], "plans", self._plans)
        key = (flavour, _lib.current_physics())
        hit = cache.get(key)
        if hit is not None:
            return hit
        lib = _lib.load()
        s = self.shape
        flux = (ctypes.c_void_p * 3)(*[b.tensor.data_ptr() for b in self.flux] + [None] * (3 - s.dim))
        lam = (ctypes.c_void_p * 3)(*[b.tensor.data_ptr() for b in self.lam] + [None] * (3 - s.dim))
        h = ctypes.c_void_p()
        _lib.check(lib.fvb_plan_create_ext(flavour, s.dim, s.patch_size, s.patch_count, 1, flux, lam,
                                           ctypes.byref(h)))
        plan = _PlanHandle(h)
        cache[key] = plan
        return plan


class _PlanHandle:
    def __init__(self, handle: ctypes.c_void_p) -> None:
        self.handle = handle
        self._fin = weakref.finalize(self, _destroy_plan, handle.value)


def _destroy_plan(h) -> None:
    if h:
        try:
            _lib.load().fvb_plan_destroy(ctypes.c_void_p(h))
        except Exception:  # pragma: no cover
            pass


class DeviceArena:
    """Device buffer source with recycling and allocation accounting
    (memory.py:105-137): ``allocate`` always creates, ``acquire`` reuses a
    recycled buffer of the same role."""

    def __init__(self, device="cuda") -> None:
        self.device = device
        self.allocation_count = 0
        self.outstanding_bytes = 0
        self.high_water_bytes = 0
        self._pool: dict[tuple, list] = {}

    def allocate(self, count: int, lazy: bool = False):
        if lazy:
            buf = _LazyBuffer(count, self.device)
        else:
            import torch

            buf = torch.empty(count, dtype=torch.float64, device=self.device)
        self.allocation_count += 1
        self.outstanding_bytes += count * 8
        self.high_water_bytes = max(self.high_water_bytes, self.outstanding_bytes)
        return buf

    def free(self, buf) -> None:
        self.outstanding_bytes -= buf.numel() * 8

    def acquire(self, key: tuple, count: int, lazy: bool = False):
        stack = self._pool.get(key)
        return stack.pop() if stack else self.allocate(count, lazy)

    def recycle(self, key: tuple, buf) -> None:
        self._pool.setdefault(key, []).append(buf)


@dataclass
class LaunchBuffers:
    """Everything one launch addresses, plus how to give it back (memory.py:140-150)."""

    mode: TransferMode
    shape: BatchShape
    layout: Layout
    batch: DeviceBatch | None
    scratch: GpuScratchArrays
    input_view: object
    output_view: object
    pooled: list = field(default_factory=list)
    owned: list = field(default_factory=list)


def _scratch_keys(shape: BatchShape, layout: Layout) -> list[tuple]:
    s = (shape.dim, shape.patch_size, shape.patch_count, layout.value)
    return [("flux", a) + s for a in range(shape.dim)] + [("lambda", a) + s for a in range(shape.dim)]


def acquire_buffers(shape: BatchShape, layout: Layout, mode: TransferMode, arena: DeviceArena,
                    scattered) -> LaunchBuffers:
    """Batch / scratch buffers and field views of one launch (memory.py:162-228).

    SHARED has no batch buffers: the views are the per-patch arrays
    themselves (AoS; the layout only matters for the temporaries).  The
    2*d step temporaries are pooled in SHARED / POOLED and allocated lazily
    (device memory only when a cascade / graph launch uses them).
    ``scattered`` may also be a DevicePatchSet (a batch already in HBM).
    """
    if scattered.shape != shape:
        raise ShapeMismatchError(f"scattered set is {scattered.shape}, launch wants {shape}")
    nf, nl = GpuScratchArrays.sizes(shape)
    sizes = [nf] * shape.dim + [nl] * shape.dim
    pooled, owned = [], []
    if mode is TransferMode.EXPLICIT_COPY:
        sbufs = [arena.allocate(n, lazy=True) for n in sizes]
        owned += sbufs
    else:
        keys = _scratch_keys(shape, layout)
        sbufs = [arena.acquire(k, n, lazy=True) for k, n in zip(keys, sizes)]
        pooled += list(zip(keys, sbufs))
    scratch = GpuScratchArrays(shape, sbufs[:shape.dim], sbufs[shape.dim:])
    if isinstance(scattered, DevicePatchSet):  # already resident: compute in place
        return LaunchBuffers(mode, shape, scattered.input.layout, None, scratch, scattered.input,
                             scattered.output, pooled, owned)
    if mode is TransferMode.SHARED:
        return LaunchBuffers(mode, shape, layout, None, scratch, scattered.input_view(),
                             scattered.output_view(), pooled, owned)
    if mode is TransferMode.EXPLICIT_COPY:
        inp, out = arena.allocate(shape.input_size), arena.allocate(shape.output_size)
        owned += [inp, out]
    else:
        in_key = ("input", shape.dim, shape.patch_size, shape.patch_count, layout.value)
        out_key = ("output",) + in_key[1:]
        inp, out = arena.acquire(in_key, shape.input_size), arena.acquire(out_key, shape.output_size)
        pooled += [(in_key, inp), (out_key, out)]
    batch = DeviceBatch(shape, layout, DeviceFieldView(inp, shape, True, layout),
                        DeviceFieldView(out, shape, False, layout))
    return LaunchBuffers(mode, shape, layout, batch, scratch, batch.input, batch.output, pooled,
                         owned)


def release_buffers(buffers: LaunchBuffers, arena: DeviceArena) -> None:
    for key, buf in buffers.pooled:
        arena.recycle(key, buf)
    for buf in buffers.owned:
        arena.free(buf)
    buffers.pooled, buffers.owned = [], []


def _stream(device=None):
    import torch

    return torch.cuda.current_stream(device)


def gather_patches(src: ScatteredPatchSet, dst: DeviceBatch) -> None:
    """Per-patch host AoS inputs -> the device batch's layout (memory.py:240-251):
    one table-gather kernel (zero-copy reads of the pinned / registered
    arrays), stream-ordered on the current stream."""
    if src.shape != dst.shape:
        raise ShapeMismatchError(f"gather from {src.shape} into {dst.shape}")
    s = dst.shape
    st = _stream(dst.input.tensor.device)
    with src.addressable(st.synchronize):  # the table and a transient registration end here
        tab = src.input_view().device_table(dst.input.tensor.device)
        _lib.check(_lib.load().fvb_gather_table(s.dim, s.patch_size, s.patch_count, 0, s.patch_count,
                                                tab.data_ptr(), LAYOUT_CODES[dst.layout],
                                                dst.input.data_ptr(), st.cuda_stream))
        st.synchronize()


def scatter_results(src: DeviceBatch, dst: ScatteredPatchSet) -> None:
    """The device batch's interior output -> per-patch host AoS outputs
    (memory.py:254-265): one table-scatter kernel (zero-copy writes)."""
    if src.shape != dst.shape:
        raise ShapeMismatchError(f"scatter from {src.shape} into {dst.shape}")
    s = src.shape
    st = _stream(src.output.tensor.device)
    with dst.addressable(st.synchronize):
        tab = dst.output_view().device_table(src.output.tensor.device)
        _lib.check(_lib.load().fvb_scatter_table(s.dim, s.patch_size, s.patch_count, 0, s.patch_count,
                                                 LAYOUT_CODES[src.layout], src.output.data_ptr(),
                                                 tab.data_ptr(), st.cuda_stream))
        st.synchronize()


# ---------------------------------------------------------------------------
# persistence: the reference's batch file (patchdata.py:337-366)
# ---------------------------------------------------------------------------
_LAYOUT_FROM_CODE = {v: k for k, v in LAYOUT_CODES.items()}


def write_batch_file(path, shape: BatchShape, layout: Layout, inp: np.ndarray, out: np.ndarray) -> None:
    """(d, p, N, T, layout) little-endian int32 header, then the input and the
    output doubles (little-endian) -- byte-compatible with the reference's
    dump_batch, so either side reads the other's files."""
    if np.size(inp) != shape.input_size or np.size(out) != shape.output_size:
        raise ShapeMismatchError("arrays do not match the batch shape")
    header = struct.pack("<5i", shape.dim, shape.patch_size, shape.unknowns, shape.patch_count,
                         LAYOUT_CODES[layout])
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(inp, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(out, dtype="<f8").tobytes())


def read_batch_file(path) -> tuple[BatchShape, Layout, np.ndarray, np.ndarray]:
    """Inverse of write_batch_file (the reference's load_batch checks)."""
    with open(path, "rb") as f:
        d, p, n, t, code = struct.unpack("<5i", f.read(20))
        shape = BatchShape(d, p, t)
        if n != shape.unknowns:
            raise ValueError(f"header unknown count {n} != d+2 = {shape.unknowns}")
        raw = f.read()
    expected = (shape.input_size + shape.output_size) * 8
    if len(raw) != expected:
        raise ValueError(f"payload of {len(raw)} bytes, expected {expected}")
    if code not in _LAYOUT_FROM_CODE:
        raise ValueError(f"unknown layout code {code}")
    data = np.frombuffer(raw, dtype="<f8")
    return (shape, _LAYOUT_FROM_CODE[code], data[: shape.input_size].astype(np.float64),
            data[shape.input_size:].astype(np.float64))


def dump_batch(batch: DeviceBatch, path) -> None:
    """Write a device batch in the reference's file format (dump_batch,
    patchdata.py:337-351): one device-to-host copy per array."""
    write_batch_file(path, batch.shape, batch.layout, batch.input.tensor.cpu().numpy(),
                     batch.output.tensor.cpu().numpy())


def load_batch(path, device="cuda") -> DeviceBatch:
    """Read a batch file (the reference's load_batch, patchdata.py:354-366)
    straight into HBM, in the file's layout."""
    import torch

    shape, layout, inp, out = read_batch_file(Path(path))
    return DeviceBatch(shape, layout,
                       DeviceFieldView(torch.from_numpy(inp).to(device), shape, True, layout),
                       DeviceFieldView(torch.from_numpy(out).to(device), shape, False, layout))
