# GPU pass: run_launch tests + bench (device + e2e only)
TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.e2e.log
timeout 900 python -m pytest tests/test_gpu_launch.py tests/test_bench.py tests/test_gpu_physics.py -x -q -m gpu > $LOG 2>&1
echo "tests rc=$?" >> $LOG
timeout 600 python bench.py --no-cpu --no-extras --no-exhaustive > gpurun_out/$TAG.bench.json 2> gpurun_out/$TAG.bench.err
echo "bench rc=$?" >> $LOG
tail -8 $LOG
python -c "
import json;d=json.load(open('gpurun_out/$TAG.bench.json'));e=d['e2e']
print('value',d['value'],'frac',d['roofline']['frac'],'clk',d['clocks'])
print('e2e',e['value'],e['mean_split_s'],e['h2d_gbs_achieved'],e['pcie_h2d_gbs_this_box'])"
