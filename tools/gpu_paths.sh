#!/bin/bash
# Secondary bench paths on one GPU: NCCL/distributed code path with one rank, streaming windows, reference arm.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config dsv3 --dist-path --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err; tail -c 400 gpurun_out/bench_dist.json; tail -3 gpurun_out/bench_dist.err
timeout 900 python bench.py --config stream --steps 3 --warmup 3 > gpurun_out/bench_stream.json 2> gpurun_out/bench_stream.err; tail -c 600 gpurun_out/bench_stream.json; tail -3 gpurun_out/bench_stream.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
