#!/bin/bash
# Iteration loop on the GPU box: parity tests of the counting paths, full GPU suite, bench + ncu for $CONFIGS.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stack or mma or stats" > gpurun_out/pytest_count.log 2>&1; tail -15 gpurun_out/pytest_count.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-dsv2lite}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
r=d['roofline']; print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r['launch_ms'],3), 'ms', r.get('tensor_ceiling',{}).get('frac'), r.get('atomic_ceiling',{}).get('frac'))"
done
if [ "${PROFILE:-1}" = "1" ]; then TAG=${TAG:-r1c} CONFIGS="${CONFIGS:-dsv2lite}" bash tools/gpu_profile_all.sh; fi
