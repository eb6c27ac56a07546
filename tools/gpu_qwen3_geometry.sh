#!/bin/bash
# Qwen3 counter geometry: 2 pairs / 2 CTAs per SM (shipped) vs 4 pairs / 1 CTA per SM (ab/q4_p4.so):
# parity tests of the i8 counters with the variant, count time (bench) and DRAM bytes (ncu).
set -u
mkdir -p gpurun_out/geo
GIMBAL_LIB=$PWD/ab/q4_p4.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "128 or qwen3" 2>&1 | tail -1
for rep in 1 2; do for lib in shipped q4_p4; do
  [ $lib = shipped ] && L="" || L=$PWD/ab/$lib.so
  env ${L:+GIMBAL_LIB=$L} timeout 600 python bench.py --config qwen3 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qwen3 $lib step', round(d['ms_per_step'],3), 'count', round(d['roofline']['launch_ms'],3))"
done; done
for lib in shipped q4_p4; do
  [ $lib = shipped ] && L="" || L=$PWD/ab/$lib.so
  env ${L:+GIMBAL_LIB=$L} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:count_mma -s 3 -c 1 --csv \
    python bench.py --config qwen3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/geo/$lib.csv 2>/dev/null
  echo "$lib: $(grep -E 'dram__bytes_read|gpu__time_duration|tensor_cycles' gpurun_out/geo/$lib.csv | awk -F'","' '{printf "%s=%s %s  ", $(NF-2), $NF, $(NF-1)}')"
done
