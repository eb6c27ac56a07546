#!/bin/bash
# Qwen3 counter (4 pairs per group) check: every i8-counter parity test, the bench line, and a
# --set full capture of the counting kernel.
set -u
O=gpurun_out/qwen3_r2e
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_engines.py tests/test_c_host.py tests/test_gpu_distributed.py -m gpu -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
timeout 900 python bench.py --config qwen3 > $O/bench_qwen3.log 2>&1; grep '^{' $O/bench_qwen3.log | tail -1 > $O/bench_qwen3.json; cut -c1-160 $O/bench_qwen3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_mma -s 3 -c 1 -o $O/count_r2e_qwen3 -f \
  python bench.py --config qwen3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/count_r2e_qwen3.ncu-rep > $O/ncu_count_r2e_qwen3.txt 2>&1; head -4 $O/ncu_count_r2e_qwen3.txt; grep tensor_cycles $O/ncu_count_r2e_qwen3.txt
