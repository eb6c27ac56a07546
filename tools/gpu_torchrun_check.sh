#!/bin/bash
# The driver's launch forms at N = 1: torchrun for both arms, and the multi-rank code path on a
# one-rank NCCL group (--dist-path), small step counts.
set -u
mkdir -p gpurun_out/torchrun
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun/ours.log 2>&1; echo "ours rc=$?"; grep '^{' gpurun_out/torchrun/ours.log | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun/ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/torchrun/ref.log | cut -c1-200
timeout 900 python bench.py --dist-path --steps 3 --warmup 3 > gpurun_out/torchrun/dist.log 2>&1; echo "dist-path rc=$?"; grep '^{' gpurun_out/torchrun/dist.log | cut -c1-200
timeout 900 python bench.py --config stream --dist-path --steps 2 --warmup 3 > gpurun_out/torchrun/dist_stream.log 2>&1; echo "dist-path stream rc=$?"; grep '^{' gpurun_out/torchrun/dist_stream.log | cut -c1-200
