import torch, statistics, sys
sys.path.insert(0, '.')
import paper_2306_16731_b200 as fvb
from paper_2306_16731_b200 import _lib
lib = fvb.load_library(); ctx = fvb.default_context()
d, p, t = 3, 8, 100_000
shape = fvb.BatchShape(d, p, t)
soa = fvb.init_field_device(shape, 0)
out = torch.empty(shape.output_size, dtype=torch.float64, device="cuda")
lam = torch.empty(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for layout in (fvb.Layout.SOA, fvb.Layout.AOS, fvb.Layout.AOSOA):
    q = fvb.relayout(soa, layout)
    for v in (0, 5):
        with _lib.tuning(_lib.FVB_TUNE_SLAB_VARIANT, v):
            ts = []
            for i in range(25):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                _lib.check(lib.fvb_step_layout(_lib.FVB_FUSED, fvb.LAYOUT_CODES[layout], d, p, t, q.data_ptr(), out.data_ptr(), ctx.dt, ctx.h, ctx.params.gamma, 1, lam.data_ptr(), None, st))
                b.record()
                if i >= 5: ts.append((a, b))
            torch.cuda.synchronize()
        print(layout.value, "variant", v, "%.1f us" % (1e3 * statistics.mean(a.elapsed_time(b) for a, b in ts)), float(lam.item()), flush=True)
