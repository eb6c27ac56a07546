#!/bin/bash
# Full GPU suite, then a short bench line per config (device value, count kernel, launches).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in ${CONFIGS:-mixtral dsv2lite qwen3 dsv3}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; count', round(r['launch_ms'],4), 'launches', d.get('gpu_launches'))" || tail -5 gpurun_out/b_$c.err
done
