#!/bin/bash
# Round-2f captures: launch lists of the Mixtral and streaming configs, ncu --set full of the Mixtral
# event-histogram counter.
set -u
O=gpurun_out/r2f
mkdir -p $O
for c in mixtral stream; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r2f_$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $O/launches_r2f_$c.log 2>&1
  python tools/launch_summary.py $O/launches_r2f_$c.csv > $O/launches_r2f_$c.md 2>&1; head -30 $O/launches_r2f_$c.md
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_events8 -s 3 -c 1 \
  -o $O/count_r2f_mixtral -f \
  python bench.py --config mixtral --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_mixtral.log 2>&1
python tools/ncu_summary.py $O/count_r2f_mixtral.ncu-rep > $O/ncu_count_r2f_mixtral.txt 2>&1
cat $O/ncu_count_r2f_mixtral.txt | head -60
