#!/bin/bash
# Full check on one GPU: GPU tests, smoke, bench lines for every config (+ stream, dist path), launch lists.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in ${CONFIGS:-dsv3 qwen3 dsv2lite mixtral stream}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 ${BENCH_EXTRA:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
e=d.get('e2e') or {}
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r.get('launch_ms',0),3), 'e2e', round(e.get('value',0)/1e6,1))" || tail -3 gpurun_out/bench_$c.err
done
if [ "${DIST:-1}" = "1" ]; then
  timeout 600 python bench.py --config dsv3 --dist-path --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_dist.json').read().strip().splitlines()[-1]); print('dist-path', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_dist.err
fi
if [ "${LAUNCHES:-0}" = "1" ]; then
  for c in ${LCONFIGS:-dsv3}; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches $c done"
  done
fi
