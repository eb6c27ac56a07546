#!/bin/bash
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
timeout 900 python -m pytest tests/test_gpu_tiny_pass.py -q -x 2>&1 | tail -3
GIMBAL_LIB=$AB timeout 300 python tools/tiny_profile.py 4096
GIMBAL_LIB=$AB timeout 300 python tools/tiny_profile.py 1
for c in mixtral dsv2lite; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; count', round(r['launch_ms'],4), 'launches', d.get('gpu_launches'))" || tail -5 gpurun_out/b_$c.err
done
