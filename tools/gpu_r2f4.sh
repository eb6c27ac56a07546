#!/bin/bash
# A/B of the small-batch online iteration: graph (count + finish kernels, stream sync) vs one fused
# launch with a host poll, ids read zero-copy (FUSED=1) or staged through shared memory (FUSED=2).
set -u
O=gpurun_out/r2f4
mkdir -p $O
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for rep in 1 2; do
  for v in graph 1 2; do
    if [ $v = graph ]; then LD_PRELOAD=$AB ./tools/microbench/online_latency 2000 > $O/lat_${v}_$rep.jsonl 2>&1
    else GIMBAL_ONLINE_FUSED=$v LD_PRELOAD=$AB ./tools/microbench/online_latency 2000 > $O/lat_${v}_$rep.jsonl 2>&1; fi
    grep '"tokens": 64' $O/lat_${v}_$rep.jsonl | sed "s/^/$v: /" | cut -c1-120
  done
done
GIMBAL_LIB=$AB GIMBAL_ONLINE_FUSED=1 timeout 600 python -m pytest tests/test_gpu_hook.py -x -q 2>&1 | tail -1
