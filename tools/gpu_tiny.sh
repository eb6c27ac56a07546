#!/bin/bash
# Fused small-shape pass: parity tests, Mixtral bench (fused vs AB unfused), launch list.
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
timeout 900 python -m pytest tests/test_gpu_tiny_pass.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_engines.py -q -x -k "unfused or alternate" 2>&1 | tail -2
for rep in 1 2; do
  for v in fused unfused; do
    if [ $v = unfused ]; then export GIMBAL_LIB=$AB GIMBAL_NO_TINY_PASS=1; else unset GIMBAL_LIB GIMBAL_NO_TINY_PASS; fi
    timeout 300 python bench.py --config mixtral --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/mx.json 2> gpurun_out/mx.err
    python -c "
import json; d=json.loads(open('gpurun_out/mx.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v mixtral', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; count', round(r['launch_ms'],4), 'launches', d.get('gpu_launches'))" || tail -3 gpurun_out/mx.err
  done
done
unset GIMBAL_LIB GIMBAL_NO_TINY_PASS
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv \
  python bench.py --config mixtral --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/mx_launches.csv 2> gpurun_out/mx_launches.err
grep -v '^{' gpurun_out/mx_launches.csv | grep -v '^==' > gpurun_out/mx_launches_clean.csv
python tools/launch_summary.py gpurun_out/mx_launches_clean.csv
