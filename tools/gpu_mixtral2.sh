#!/bin/bash
# Mixtral: lane-private vs shared-table counting (AB build), then the per-kernel launch list of the
# graph-replayed step (warm caches) to see where the step's time goes.
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "lanepriv or stats or small" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_engines.py -q -x -k "alternate_counters" 2>&1 | tail -2
for rep in 1 2; do
  for v in 1 0; do
    GIMBAL_LIB=$AB GIMBAL_SMALL_SHARED=$v timeout 300 python bench.py --config mixtral --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/mx.json 2> gpurun_out/mx.err
    python -c "
import json; d=json.loads(open('gpurun_out/mx.json').read().strip().splitlines()[-1]); r=d['roofline']
print('shared=$v mixtral', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; count', round(r['launch_ms'],4), r.get('kernel'))" || tail -3 gpurun_out/mx.err
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
  python bench.py --config mixtral --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/mx_launches.csv 2> gpurun_out/mx_launches.err
python tools/launch_summary.py gpurun_out/mx_launches.csv
