"""A/B of fused-kernel launch shapes on one config (device time, L2 flushed).

    python scripts/small_ab.py --dim 2 --p 3 --patches 100000 --variants 0,6

Each variant is an FVB_TUNE_PENCIL_VARIANT (2D) / FVB_TUNE_SLAB_VARIANT (3D)
value; reduce filter default.  Prints one line per variant: mean / min ms,
cell updates/s, fraction of the HBM roofline, and checks every variant's
output and eigenvalue equal the first's.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--patches", type=int, default=100_000)
    ap.add_argument("--variants", default="0,6")
    ap.add_argument("--filter", type=int, default=-1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--flush", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2306_16731_b200 as fvb
    from paper_2306_16731_b200 import _lib

    lib = fvb.load_library()
    ctx = fvb.default_context()
    shape = fvb.BatchShape(a.dim, a.p, a.patches)
    q = fvb.init_field_device(shape, 0)
    out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
    lam = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda") if a.flush else None
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda") if a.flush else None
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    nbytes = a.patches * 8 * (a.dim + 2) * ((a.p + 2) ** a.dim + a.p ** a.dim)
    key = _lib.FVB_TUNE_PENCIL_VARIANT if a.dim == 2 else _lib.FVB_TUNE_SLAB_VARIANT
    ref = None
    for v in [int(x) for x in a.variants.split(",")]:
        with _lib.tuning(key, v), _lib.tuning(_lib.FVB_TUNE_REDUCE_FILTER, a.filter):
            ts = []
            for i in range(a.steps + 5):
                if flush is not None:
                    flush.fill_(float(i))
                    if a.flush == 2:  # read another 256 MB: the L2 left clean (no dirty write-backs)
                        clean.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                _lib.check(lib.fvb_step(_lib.FVB_FUSED, a.dim, a.p, a.patches, q.data_ptr(), out.data_ptr(),
                                        ctx.dt, ctx.h, ctx.params.gamma, 1, lam.data_ptr(), None, st.cuda_stream))
                e1.record(st)
                if i >= 5:
                    ts.append((e0, e1))
            torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ts]
        mean = statistics.mean(ms)
        got = (out.clone(), float(lam.item()))
        same = ref is None or (torch.equal(got[0], ref[0]) and got[1] == ref[1])
        ref = ref or got
        print(f"variant {v}: mean {mean*1e3:.1f} us  min {min(ms)*1e3:.1f} us  "
              f"{a.patches * a.p ** a.dim / (mean * 1e-3):.3e} cell/s  frac {nbytes / (mean * 1e-3) / 1e9 / peak:.3f}  "
              f"same={same}", flush=True)


if __name__ == "__main__":
    main()
