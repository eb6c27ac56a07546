#!/bin/bash
# Round-2f measurement at HEAD: full GPU suite, smoke, every bench config (device value, e2e, CPU
# baseline), the reference arm, the online hook latency (Python and C), launch lists, and a --set full
# capture of the Mixtral event counter (the DS-V3 counter is unchanged since profiles/r2e/).
set -u
O=gpurun_out/final_r2f
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for c in dsv3 mixtral dsv2lite qwen3 stream; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.log 2>&1
  grep '^{' $O/bench_$c.log | tail -1 > $O/bench_$c.json
  python -c "
import json; d=json.load(open('$O/bench_$c.json')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; e2e', round((e.get('value') or 0)/1e6,1), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', r.get('frac'), 'clk', d.get('clocks'))" || tail -5 $O/bench_$c.log
done
timeout 1200 python bench.py --impl reference > $O/bench_reference.log 2>&1
grep '^{' $O/bench_reference.log | tail -1 > $O/bench_reference.json; cut -c1-300 $O/bench_reference.json
timeout 900 python tools/hook_latency.py --iters 300 > $O/hook_latency.jsonl 2>&1; tail -1 $O/hook_latency.jsonl | cut -c1-200
./tools/microbench/online_latency 2000 > $O/online_latency_c.jsonl 2>&1; tail -2 $O/online_latency_c.jsonl
for c in dsv3 mixtral; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r2f_$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $O/launches_r2f_$c.log 2>&1
  python tools/launch_summary.py $O/launches_r2f_$c.csv > $O/launches_r2f_$c.md 2>&1; head -6 $O/launches_r2f_$c.md
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_events8 -s 3 -c 1 \
  -o $O/count_r2f_mixtral -f python bench.py --config mixtral --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/count_r2f_mixtral.ncu-rep > $O/ncu_count_r2f_mixtral.txt 2>&1; head -4 $O/ncu_count_r2f_mixtral.txt
