#!/bin/bash
# Launch lists for every config + one ncu --set full capture of each config's counting kernel.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1b}
for c in ${CONFIGS:-dsv3 qwen3 dsv2lite mixtral}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches_${TAG}_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-count_} -s ${SKIP:-3} -c 1 \
    -o gpurun_out/count_${TAG}_$c -f \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${TAG}_$c.log 2>&1
  echo "$c done"
done
