#!/bin/bash
# Round-2e measurement: full GPU suite, smoke, every bench config (device value, e2e, CPU baseline),
# the reference arm, the online hook latency, compute-sanitizer over the kernels added in 2d/2e
# (exact_solve enumeration, eval_dev bins, the deeper eval id ring, the block-wide u16 drain), and
# a --set full capture of the DS-V3 counter.
set -u
O=gpurun_out/final_r2e
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
timeout 900 python tools/hook_latency.py --iters 200 > $O/hook_latency.jsonl 2>&1; tail -1 $O/hook_latency.jsonl | cut -c1-200
SAN_TESTS="tests/test_gpu_exact.py tests/test_gpu_parity.py::test_eval_tensor_core_path_matches_oracle tests/test_gpu_parity.py::test_eval_rejects_infeasible_candidate tests/test_gpu_engines.py::test_alternate_counters"
for tool in memcheck synccheck racecheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 200 --log-file $O/san_$tool.log \
    python -m pytest $SAN_TESTS -q -p no:cacheprovider > $O/san_${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 $O/san_${tool}_pytest.log)"; tail -1 $O/san_$tool.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_tm -s 3 -c 1 -o $O/count_r2e_dsv3 -f \
  python bench.py --config dsv3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/count_r2e_dsv3.ncu-rep > $O/ncu_count_r2e_dsv3.txt 2>&1; head -4 $O/ncu_count_r2e_dsv3.txt
