#!/bin/bash
# A/B kernel experiment on one GPU box: bench each ab/*.so build on $CONFIGS, interleaved, $REPS times.
set -u
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do
  for so in ab/*.so; do
    for c in ${CONFIGS:-dsv2lite}; do
      GIMBAL_LIB=$PWD/$so timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
      python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$so', '$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r['launch_ms'],3))" || tail -3 gpurun_out/ab.err
    done
  done
done
