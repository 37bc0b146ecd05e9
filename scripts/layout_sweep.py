"""Batch-layout comparison on one B200 (the reference's Appendix C
layout study): AoS vs SoA vs AoSoA device batches for the
fused and cascade flavours at C3's top point (2D p=16, 2^20 patches) and C4
(3D p=8, 100k patches).  Device time per step (CUDA events, mean of --steps).

    python scripts/layout_sweep.py [--out gpurun_out/layouts.csv]
"""
import argparse
import csv
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "layouts.csv"))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch
    import paper_2306_16731_b200 as fvb
    from paper_2306_16731_b200 import _lib

    lib = fvb.load_library()
    ctx = fvb.default_context()
    rows = []
    for d, p, t in ((2, 16, 1 << 20), (3, 8, 100_000)):
        shape = fvb.BatchShape(d, p, t)
        soa = fvb.init_field_device(shape, 0)
        out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
        lam = torch.empty(1, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        bytes_step = t * 8 * (d + 2) * ((p + 2) ** d + p ** d)
        ref = None
        for layout in (fvb.Layout.SOA, fvb.Layout.AOSOA, fvb.Layout.AOS):
            q = fvb.relayout(soa, layout)
            for name, fl in (("fused", _lib.FVB_FUSED), ("cascade", _lib.FVB_CASCADE)):
                def step():
                    _lib.check(lib.fvb_step_layout(fl, fvb.LAYOUT_CODES[layout], d, p, t, q.data_ptr(),
                                                   out.data_ptr(), ctx.dt, ctx.h, ctx.params.gamma, 1,
                                                   lam.data_ptr(), None, st))
                for _ in range(args.warmup):
                    step()
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(args.steps)]
                for a, b in evs:
                    a.record()
                    step()
                    b.record()
                torch.cuda.synchronize()
                ms = [a.elapsed_time(b) for a, b in evs]
                mean_s = statistics.mean(ms) * 1e-3
                red = float(lam.item())
                if ref is None:
                    ref = red
                assert red == ref, (layout, name, red, ref)  # bit-identical across layouts
                cells = t * p ** d
                rows.append(dict(dim=d, p=p, T=t, layout=layout.value, flavour=name, mean_s=mean_s,
                                 min_s=min(ms) * 1e-3, cell_updates_per_s=cells / mean_s,
                                 algo_GBps=bytes_step / mean_s / 1e9, reduced=red))
                print(f"d={d} p={p} T={t:8d} {layout.value:6s} {name:8s} {mean_s * 1e3:9.3f} ms "
                      f"{cells / mean_s / 1e9:7.2f} Gcell/s {bytes_step / mean_s / 1e9:8.1f} GB/s",
                      flush=True)
            del q
        ref = None
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    with open(args.out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)


if __name__ == "__main__":
    main()
