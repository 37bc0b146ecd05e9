# 2D AoS: 16-byte unknown-pair copies (variant 0) vs 8-byte (variant 9); parity tests first
TAG=$1
LOG=gpurun_out/$TAG.aos2d.log; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -m gpu -x -k "layout or random or acceptance or degenerate or unaligned" 2>&1 | tail -2
python - <<'PY'
import torch, statistics, sys
sys.path.insert(0, '.')
import paper_2306_16731_b200 as fvb
from paper_2306_16731_b200 import _lib
lib = fvb.load_library(); ctx = fvb.default_context()
for d, p, t in ((2, 16, 1 << 20), (2, 5, 200_000), (2, 3, 100_000)):
    shape = fvb.BatchShape(d, p, t)
    q = fvb.relayout(fvb.init_field_device(shape, 0), fvb.Layout.AOS)
    out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
    lam = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for v in (0, 9, 0, 9):
        with _lib.tuning(_lib.FVB_TUNE_PENCIL_VARIANT, v):
            ts = []
            for i in range(25):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                _lib.check(lib.fvb_step_layout(_lib.FVB_FUSED, 0, d, p, t, q.data_ptr(), out.data_ptr(), ctx.dt, ctx.h, ctx.params.gamma, 1, lam.data_ptr(), None, st))
                b.record()
                if i >= 5: ts.append((a, b))
            torch.cuda.synchronize()
        print(f"d={d} p={p} T={t} aos variant {v}: {statistics.mean(a.elapsed_time(b) for a, b in ts):.3f} ms  lam {float(lam.item())!r}", flush=True)
PY
} > $LOG 2>&1
cat $LOG
