#!/bin/bash
# Profiling recipe (under gpurun, 1 GPU): launch list of one bench step + one ncu --set full
# capture of the dominant kernel.  Usage: tools/gpu_profile.sh <tag> [config] [tokens]
set -u
TAG=${1:-r1}; CFG=${2:-dsv3}; TOK=${3:-0}
mkdir -p gpurun_out
EXTRA=""
[ "$TOK" != "0" ] && EXTRA="--tokens $TOK"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:count_ -s 3 -c 1 \
    -o gpurun_out/count_${TAG}_${CFG} -f \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/ncu_${TAG}_${CFG}.log 2>&1
echo "profile done: $TAG $CFG"
