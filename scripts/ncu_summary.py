"""Summarise an .ncu-rep: key metrics + executed-opcode histogram (per cell) + stall top list.
usage: python scripts/ncu_summary.py REP CELLS_PER_LAUNCH"""
import collections, csv, io, subprocess, sys

rep, cells = sys.argv[1], float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
d = dict(zip(h, rows[2]))
keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
        v = float(d[k] or 0)
        if v > 0.05:
            print(f"{k:70s} {v:.3f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc, iss = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ia])
    except (ValueError, IndexError):
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    cnt[o] += n
    stall[o] += int(r[iss] or 0)
tot = sum(cnt.values())
print(f"total warp inst {tot}  per cell (thread-level) {tot * 32 / cells:.1f}")
fp64 = sum(v for k, v in cnt.items() if k.startswith(("DADD", "DMUL", "DFMA", "DSETP", "DMNMX")))
print(f"fp64 per cell {fp64 * 32 / cells:.1f}")
for k, v in cnt.most_common(40):
    print(f"  {k:22s} {v * 32 / cells:8.2f}/cell  stall-samples {stall[k]}")
