#!/bin/bash
# Mixtral event counter with both layers of a row word canonicalised at once (u16x2 min/max): full
# GPU suite, the Mixtral bench line, and a --set full capture of the counter.
set -u
O=gpurun_out/r2f8
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py --config mixtral 2>/dev/null | grep '^{' | tail -1 > $O/bench_mixtral.json
python -c "import json; d=json.load(open('$O/bench_mixtral.json')); print('mixtral', d['ms_per_step'], d['roofline']['launch_ms'], d['e2e']['value']/1e6, d['cpu_baseline']['value']/1e6)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_events8 -s 3 -c 1 \
  -o $O/count_r2f8_mixtral -f python bench.py --config mixtral --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/count_r2f8_mixtral.ncu-rep > $O/ncu_count_r2f8_mixtral.txt 2>&1; grep -E "duration|inst_executed.sum|stall" $O/ncu_count_r2f8_mixtral.txt
