#!/bin/bash
# DS-V3 counter: one ncu --set full capture each of the rolling (AB) and block-wide drains, raw pages
# exported for a metric diff (profiles/r2c_dsv3_drain_traffic.md).
set -u
mkdir -p gpurun_out/drain
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for v in roll sync; do
  if [ $v = roll ]; then export GIMBAL_U15_ROLLING=1; else unset GIMBAL_U15_ROLLING; fi
  env GIMBAL_LIB=$AB timeout 900 ncu --set full --clock-control none -k regex:count_tm -s 3 -c 1 -o gpurun_out/drain/$v -f \
    python bench.py --config dsv3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/drain/$v.log 2>&1
  ncu -i gpurun_out/drain/$v.ncu-rep --page raw --csv > gpurun_out/drain/$v.raw.csv 2>&1
done
ls -la gpurun_out/drain
