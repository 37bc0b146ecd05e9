"""Streamed host->device->host step: transfers overlapped with compute (f1 row).

The paper observes that runtimes are dominated by data transfers when the
patches live on the host.  The reference emulates the
transfer modes with a gather / compute / scatter sequence
(pkg/src/patchbench/bench.py:222-258, memory.py:240-265).  On B200 the
same launch is pipelined over patch chunks on three CUDA streams:

    H2D stream:      copy chunk c's pinned AoS block into device slot c%2
    compute stream:  AoS->SoA permute, fused step on the chunk, SoA->AoS
    D2H stream:      copy chunk c's AoS result back into the pinned output

so the PCIe copies in both directions (full duplex) overlap each other and
the kernels; the step itself is bit-identical to the one-shot launch
because patches are independent (no cross-patch DAG edges,
kernelgraph.py:215-247).  Each chunk reduces into its own eigenvalue slot;
the batch value is the max of the slots (exact).
"""

from __future__ import annotations

from . import _lib
from .context import TimeStepContext
from .memory import ScatteredPatchSet
from .patchdata import BatchShape

__all__ = ["StreamedStep"]


class StreamedStep:
    """Pipelined H2D / step / D2H over ``chunks`` patch chunks (2 device slots)."""

    def __init__(self, shape: BatchShape, chunks: int = 8, flavour: int = _lib.FVB_FUSED,
                 device="cuda") -> None:
        import torch

        self.shape = shape
        self.chunks = max(1, min(int(chunks), shape.patch_count))
        self.flavour = flavour
        self.device = torch.device(device)
        t = shape.patch_count
        base, rem = divmod(t, self.chunks)
        self.bounds = []
        lo = 0
        for c in range(self.chunks):
            hi = lo + base + (1 if c < rem else 0)
            self.bounds.append((lo, hi))
            lo = hi
        tmax = base + (1 if rem else 0)
        nin = shape.unknowns * shape.haloed_cells
        nout = shape.unknowns * shape.interior_cells
        self.nin, self.nout = nin, nout
        f64 = dict(dtype=torch.float64, device=self.device)
        self.slots = [dict(in_aos=torch.empty(tmax * nin, **f64),
                           in_soa=torch.empty(tmax * nin, **f64),
                           out_soa=torch.empty(tmax * nout, **f64),
                           out_aos=torch.empty(tmax * nout, **f64)) for _ in range(2)]
        self.lam = torch.zeros(self.chunks, **f64)
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.ev_h2d = [ev() for _ in range(self.chunks)]
        self.ev_comp = [ev() for _ in range(self.chunks)]
        self.ev_in_free = [ev() for _ in range(self.chunks)]
        self.ev_out_free = [ev() for _ in range(self.chunks)]
        self.kernel_launches_per_step = 3 * self.chunks  # permute, step, permute

    def bytes_per_step(self) -> tuple[int, int]:
        s = self.shape
        return s.input_size * 8, s.output_size * 8 + 8

    def run(self, host_in, host_out, ctx: TimeStepContext, with_reduction: bool = True):
        """Enqueue one streamed step.  host_in / host_out: pinned float64 CPU
        tensors holding the concatenated per-patch AoS arrays.  Returns the
        device tensor of per-chunk eigenvalue slots (max them for the batch)."""
        import torch

        lib = _lib.load()
        d, p = self.shape.dim, self.shape.patch_size
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.wait_stream(cur)
        for c, (lo, hi) in enumerate(self.bounds):
            slot = self.slots[c % 2]
            tc = hi - lo
            with torch.cuda.stream(self.s_h2d):
                if c >= 2:
                    self.s_h2d.wait_event(self.ev_in_free[c - 2])
                slot["in_aos"][:tc * self.nin].copy_(host_in[lo * self.nin:hi * self.nin],
                                                     non_blocking=True)
                self.ev_h2d[c].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_h2d[c])
                if c >= 2:
                    self.s_comp.wait_event(self.ev_out_free[c - 2])
                st = self.s_comp.cuda_stream
                _lib.check(lib.fvb_aos_to_soa(d, p, tc, 1, slot["in_aos"].data_ptr(),
                                              slot["in_soa"].data_ptr(), st))
                self.ev_in_free[c].record(self.s_comp)
                lam_ptr = self.lam[c:c + 1].data_ptr() if with_reduction else None
                _lib.check(lib.fvb_step(self.flavour, d, p, tc, slot["in_soa"].data_ptr(),
                                        slot["out_soa"].data_ptr(), ctx.dt, ctx.h,
                                        ctx.params.gamma, int(with_reduction), lam_ptr, None, st))
                _lib.check(lib.fvb_soa_to_aos(d, p, tc, 0, slot["out_soa"].data_ptr(),
                                              slot["out_aos"].data_ptr(), st))
                self.ev_comp[c].record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(self.ev_comp[c])
                host_out[lo * self.nout:hi * self.nout].copy_(slot["out_aos"][:tc * self.nout],
                                                              non_blocking=True)
                self.ev_out_free[c].record(self.s_d2h)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            cur.wait_stream(s)
        return self.lam

    def run_scattered(self, patches: ScatteredPatchSet, ctx: TimeStepContext,
                      with_reduction: bool = True) -> float | None:
        """Blocking convenience form on a pinned ScatteredPatchSet."""
        import torch

        if patches.in_block is None or patches.out_block is None:
            raise ValueError("StreamedStep needs a contiguous (allocate_scattered) patch set")
        lam = self.run(torch.from_numpy(patches.in_block), torch.from_numpy(patches.out_block),
                       ctx, with_reduction)
        torch.cuda.current_stream(self.device).synchronize()
        return max(0.0, float(lam.max().item())) if with_reduction else None
