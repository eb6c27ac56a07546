#!/bin/bash
# Mixtral step composition: kernel launch list (ncu, one step after warm-up) + bench timing.
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mixtral.csv \
  python bench.py --config mixtral --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches_mixtral.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_mixtral.csv 2>&1 | tail -30
for i in 1 2; do timeout 300 python bench.py --config mixtral --steps 50 --warmup 10 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mixtral', d['ms_per_step'], d['roofline']['launch_ms'])"; done
