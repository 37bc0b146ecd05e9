"""Multi-step loop cost per step: host-dt loop (one eigenvalue
read per step) vs device-dt loop vs the same steps replayed as one CUDA graph.

    python scripts/multistep_bench.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2306_16731_b200.simulation import PatchGridSimulation

    for d, p, grid in ((2, 16, (8, 8)), (2, 16, (64, 64)), (2, 3, (100, 100)), (3, 8, (4, 4, 4))):
        k = 200
        res = {}
        for mode in ("host", "device", "graph"):
            sim = PatchGridSimulation(d, p, grid, seed=1)
            if mode == "graph":
                sim.capture(k)
                sim.replay()
            else:
                for _ in range(10):
                    sim.step() if mode == "host" else sim.step_device()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode == "host":
                for _ in range(k):
                    sim.step()
            elif mode == "device":
                sim.run_device(k)
            else:
                sim.replay()
            torch.cuda.synchronize()
            res[mode] = (time.perf_counter() - t0) / k * 1e6
        print(f"d={d} p={p} grid={grid}: us/step host-dt {res['host']:.1f}, device-dt "
              f"{res['device']:.1f}, CUDA graph {res['graph']:.1f}", flush=True)


if __name__ == "__main__":
    main()
