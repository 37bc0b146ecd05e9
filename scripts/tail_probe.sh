# C2 work quantisation / fixed cost: tile-kernel device time vs patch count
# (148 SMs x 5 CTAs x 32-patch groups = 23680 patches per round), beside a
# trivial kernel timed the same way.
TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.tail.log
{
python - <<'PY'
import torch, statistics
x = torch.zeros(1, device="cuda"); fl = torch.empty(64 << 20, device="cuda"); cl = torch.ones(64 << 20, device="cuda")
st = torch.cuda.current_stream(); ts = []
for i in range(45):
    fl.fill_(float(i)); cl.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); x.add_(1.0); b.record(st)
    if i >= 5: ts.append((a, b))
torch.cuda.synchronize()
print("trivial kernel (x.add_) event time: mean %.1f us" % (1e3 * statistics.mean(a.elapsed_time(b) for a, b in ts)))
PY
for T in 32 3200 23680 47360 71040 94720 100000 118400; do
  echo -n "T=$T: "; timeout 120 python scripts/small_ab.py --p 3 --patches $T --variants 0 --flush 2 --steps 40 | tail -1
done
} > $LOG 2>&1
cat $LOG
