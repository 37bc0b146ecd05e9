"""BASELINE configs[1..3] on one GPU: patch-count sweep of the three flavours.

    python scripts/flavour_sweep.py [--out profiles/flavours.csv]

configs[2]: 2D p=16, T = 2^10 .. 2^20, cascade vs fused (nested) vs CUDA-graph;
configs[1]: 2D p=3, T = 100k, all three flavours;
configs[3]: 3D p=8, T = 100k, all three flavours.
Device time per step (CUDA events, mean of --steps after --warmup), cell
updates/s and algorithmic HBM GB/s.  Inputs are the seeded field in HBM;
batches smaller than 512 MB run with a clean, cold L2 (256 MB written,
256 MB read before every step), larger ones exceed the 126 MB L2 anyway.
"""
import argparse
import csv
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def flavour_bytes(name: str, d: int, p: int) -> int:
    """HBM bytes per patch each flavour must move (its own roofline numerator).

    fused: read the haloed input once, write the output once (algorithmic).
    cascade / graph (one kernel per reference step, scratch in HBM):
      copy     read + write N*p^d
      flux_a   read + write N*R      (R = (p+2)*p^(d-1), the axis range)
      lambda_a read N*R, write R
      acc_a    read Q N*R, F N*R, lambda R; read + write the output N*p^d
      reduce   read N*p^d
    """
    n, m, pi, r = d + 2, (p + 2) ** d, p ** d, (p + 2) * p ** (d - 1)
    if name == "fused":
        return 8 * n * (m + pi)
    per_axis = 2 * n * r + (n * r + r) + (n * r + n * r + r + 2 * n * pi)
    return 8 * (2 * n * pi + d * per_axis + n * pi)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "flavours.csv"))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch
    import paper_2306_16731_b200 as fvb
    from paper_2306_16731_b200 import _lib

    lib = fvb.load_library()
    ctx = fvb.default_context()
    cases = [(2, 16, 1 << e) for e in range(10, 21, 2)] + [(2, 16, 1 << 20), (2, 3, 100_000),
                                                           (3, 8, 100_000)]
    rows = []
    for d, p, t in cases:
        shape = fvb.BatchShape(d, p, t)
        q = fvb.init_field_device(shape, 0)
        out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
        lam = torch.empty(1, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        bytes_step = t * 8 * (d + 2) * ((p + 2) ** d + p ** d)
        small = bytes_step < (512 << 20)
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda") if small else None
        clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda") if small else None
        for name, fl in (("fused", _lib.FVB_FUSED), ("cascade", _lib.FVB_CASCADE),
                         ("graph", _lib.FVB_GRAPH)):
            def step():
                _lib.check(lib.fvb_step(fl, d, p, t, q.data_ptr(), out.data_ptr(), ctx.dt, ctx.h,
                                        ctx.params.gamma, 1, lam.data_ptr(), None, st))
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            times = []
            for _ in range(args.steps):
                if flush is not None:  # footprint < L2: clean, cold L2 before every step
                    flush.fill_(1.0)
                    clean.sum()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                step()
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b) * 1e-3)
            s = statistics.mean(times)
            cells = t * p ** d
            own = t * flavour_bytes(name, d, p)
            rows.append(dict(dim=d, p=p, T=t, flavour=name, mean_s=s, min_s=min(times),
                             cell_updates_per_s=cells / s, algo_GBps=bytes_step / s / 1e9,
                             flavour_bytes=own, flavour_GBps=own / s / 1e9,
                             reduced=float(lam.item())))
            print(f"d={d} p={p} T={t:>8} {name:8s} {s * 1e3:9.3f} ms {cells / s / 1e9:7.2f} "
                  f"Gcell/s {bytes_step / s / 1e9:8.1f} GB/s algorithmic, "
                  f"{own / s / 1e9:8.1f} GB/s of its own traffic", flush=True)
        lib.fvb_release_all()
        del q, out
        torch.cuda.empty_cache()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    with open(args.out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)


if __name__ == "__main__":
    main()
