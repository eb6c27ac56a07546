#!/bin/bash
# DS-V3 counter check after a kernel change: its GPU tests, the bench line, and one ncu --set full
# capture of the shipped counter (summary text + report under gpurun_out/r2d/).
set -u
mkdir -p gpurun_out/r2d
timeout 1200 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -k "256 or dsv3 or alternate" > gpurun_out/r2d/gputest.log 2>&1; tail -2 gpurun_out/r2d/gputest.log
timeout 900 python bench.py --config dsv3 > gpurun_out/r2d/bench_dsv3.log 2>&1
grep '^{' gpurun_out/r2d/bench_dsv3.log | tail -1 > gpurun_out/r2d/bench_dsv3.json; cut -c1-200 gpurun_out/r2d/bench_dsv3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_tm -s 3 -c 1 -o gpurun_out/r2d/count_r2d_dsv3 -f \
  python bench.py --config dsv3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2d/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2d/count_r2d_dsv3.ncu-rep > gpurun_out/r2d/ncu_count_r2d_dsv3.txt 2>&1
head -5 gpurun_out/r2d/ncu_count_r2d_dsv3.txt
