#!/bin/bash
# GPU test suite + short bench lines (default config, --dist-path, stream) + reference arm.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_dsv3.json 2> gpurun_out/bench_dsv3.err; tail -c 3000 gpurun_out/bench_dsv3.json; tail -3 gpurun_out/bench_dsv3.err
timeout 600 python bench.py --steps 5 --warmup 3 --dist-path --no-e2e --no-cpu > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err; tail -c 600 gpurun_out/bench_dist.json; tail -3 gpurun_out/bench_dist.err
