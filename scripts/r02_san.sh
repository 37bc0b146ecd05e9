# compute-sanitizer evidence + the sweep/launch API tests
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py -x -q -m gpu > gpurun_out/$TAG.api.log 2>&1; echo "api rc=$?" >> gpurun_out/$TAG.api.log
tail -3 gpurun_out/$TAG.api.log
bash scripts/sanitize.sh $TAG
