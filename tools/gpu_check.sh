#!/bin/bash
# One gpurun call: GPU parity tests, smoke, and a short bench line per config.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for c in ${CONFIGS:-dsv3 qwen3 dsv2lite mixtral}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 ${BENCH_EXTRA:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c: $(tail -c 600 gpurun_out/bench_$c.json)"
done
