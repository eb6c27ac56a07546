set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stack" > gpurun_out/pytest_stack.log 2>&1; tail -15 gpurun_out/pytest_stack.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
CONFIGS="dsv2lite" bash tools/gpu_check.sh 2>/dev/null | tail -1 | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_dsv2lite.json').read().strip().splitlines()[-1])
print(d['value']/1e6, d['ms_per_step'], d['roofline']['launch_ms'], d['roofline'].get('tensor_ceiling'))"
TAG=r1c CONFIGS=dsv2lite bash tools/gpu_profile_all.sh
