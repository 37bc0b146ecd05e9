"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently, with 1 or 2
streams per direction (what the run_launch pipeline can reach)."""
import torch


def bw(nstreams_up, nstreams_dn, nbytes=2 << 30, reps=3):
    up = [torch.empty(nbytes // 8, dtype=torch.float64).pin_memory() for _ in range(max(1, nstreams_up))]
    dn = [torch.empty(int(nbytes * 0.79) // 8, dtype=torch.float64).pin_memory() for _ in range(max(1, nstreams_dn))]
    dup = [torch.empty(nbytes // 8, dtype=torch.float64, device="cuda") for _ in range(max(1, nstreams_up))]
    ddn = [torch.empty(int(nbytes * 0.79) // 8, dtype=torch.float64, device="cuda") for _ in range(max(1, nstreams_dn))]
    su = [torch.cuda.Stream() for _ in range(nstreams_up)]
    sd = [torch.cuda.Stream() for _ in range(nstreams_dn)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for s in su + sd:
        s.wait_stream(main)
    for _ in range(reps):
        for i, s in enumerate(su):
            with torch.cuda.stream(s):
                dup[i].copy_(up[i], non_blocking=True)
        for i, s in enumerate(sd):
            with torch.cuda.stream(s):
                dn[i].copy_(ddn[i], non_blocking=True)
    for s in su + sd:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return (nstreams_up * reps * nbytes / t / 1e9, nstreams_dn * reps * int(nbytes * 0.79) / t / 1e9)


for cfg in ((1, 0), (0, 1), (1, 1), (2, 0), (2, 2), (3, 3)):
    u, d = bw(*cfg)
    print(f"streams up {cfg[0]} down {cfg[1]}: H2D {u:6.1f} GB/s  D2H {d:6.1f} GB/s  sum {u + d:6.1f}", flush=True)
