#!/bin/bash
# Round-2b measurement: full GPU suite, smoke, every bench config (device value, e2e, CPU baseline),
# the reference arm, the online hook latency.
set -u
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final/gputest.log 2>&1; tail -2 gpurun_out/final/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
for c in dsv3 mixtral dsv2lite qwen3 stream; do
  timeout 1200 python bench.py --config $c > gpurun_out/final/bench_$c.log 2>&1
  grep '^{' gpurun_out/final/bench_$c.log | tail -1 > gpurun_out/final/bench_$c.json
  python -c "
import json; d=json.load(open('gpurun_out/final/bench_$c.json')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; e2e', round((e.get('value') or 0)/1e6,1), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', r.get('frac'))" || tail -5 gpurun_out/final/bench_$c.log
done
timeout 1200 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1
grep '^{' gpurun_out/final/bench_reference.log | tail -1 > gpurun_out/final/bench_reference.json; cut -c1-300 gpurun_out/final/bench_reference.json
timeout 900 python tools/hook_latency.py --iters 200 > gpurun_out/final/hook_latency.jsonl 2>&1; tail -2 gpurun_out/final/hook_latency.jsonl | cut -c1-200
