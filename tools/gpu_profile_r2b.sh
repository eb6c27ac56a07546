#!/bin/bash
# Round-2b captures: launch list per config + ncu --set full of each config's counting kernel, and of
# the fused small-shape pass (Mixtral).  Summaries via tools/ncu_summary.py.
set -u
mkdir -p gpurun_out/r2b
TAG=r2b
for c in ${CONFIGS:-mixtral dsv2lite qwen3 dsv3}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b/launches_${TAG}_$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2b/launches_${TAG}_$c.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:count_ -s 3 -c 1 \
    -o gpurun_out/r2b/count_${TAG}_$c -f \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2b/ncu_${TAG}_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2b/count_${TAG}_$c.ncu-rep > gpurun_out/r2b/ncu_count_${TAG}_$c.txt 2>&1
  echo "$c done"; head -8 gpurun_out/r2b/ncu_count_${TAG}_$c.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiny_pass -s 3 -c 1 \
  -o gpurun_out/r2b/tiny_pass_${TAG}_mixtral -f \
  python bench.py --config mixtral --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2b/ncu_tiny.log 2>&1
python tools/ncu_summary.py gpurun_out/r2b/tiny_pass_${TAG}_mixtral.ncu-rep > gpurun_out/r2b/ncu_tiny_${TAG}_mixtral.txt 2>&1
head -8 gpurun_out/r2b/ncu_tiny_${TAG}_mixtral.txt
