#!/bin/bash
# Qwen3 tensor-core counter: rows cleared by their previous ids instead of zeroed — parity and timing.
set -u
O=gpurun_out/r2f6
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k qwen3 > $O/scale.log 2>&1; tail -1 $O/scale.log
for i in 1 2; do
  timeout 600 python bench.py --config qwen3 --no-e2e --no-cpu 2>/dev/null | grep '^{' | tail -1 > $O/bench_qwen3_$i.json
  python -c "import json; d=json.load(open('$O/bench_qwen3_$i.json')); print('qwen3', d['ms_per_step'], d['roofline'].get('launch_ms'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:count_mma -s 3 -c 1 \
  python bench.py --config qwen3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_qwen3.txt 2>&1
grep -E "duration|wavefronts|tensor|dram|inst_executed" $O/ncu_qwen3.txt | tail -5
timeout 200 python tools/fuzz_parity.py --what pass --seconds 120 > $O/fuzz_pass.log 2>&1; tail -1 $O/fuzz_pass.log
