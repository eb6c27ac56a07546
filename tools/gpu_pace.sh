#!/bin/bash
# Pacing A/B for the tensor-core counters (GIMBAL_PACE = tiles per epoch, 0 = off; AB build), then
# DRAM bytes / tensor-pipe activity of the counting kernel under ncu for off vs the default.
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
ncu --query-metrics 2>/dev/null | grep -iE 'pipe_tensor|tcgen|utc' > gpurun_out/tensor_metrics.txt
for rep in 1 2; do
  for c in ${CONFIGS:-qwen3 dsv2lite}; do
    for P in ${PACES:-0 16 64 256}; do
      GIMBAL_LIB=$AB GIMBAL_PACE=$P timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/pace.json 2> gpurun_out/pace.err
      python -c "
import json; d=json.loads(open('gpurun_out/pace.json').read().strip().splitlines()[-1]); r=d['roofline']
print('pace=$P', '$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r['launch_ms'],3))" || tail -3 gpurun_out/pace.err
    done
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
for c in ${CONFIGS:-qwen3 dsv2lite}; do
  for P in 0 ${NCU_PACE:-64}; do
    GIMBAL_LIB=$AB GIMBAL_PACE=$P timeout 900 ncu --metrics $M --clock-control none -k regex:count_ -s 3 -c 1 --csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_pace_${c}_$P.csv 2> gpurun_out/ncu_pace_${c}_$P.err
    echo "ncu $c pace=$P"; grep -E 'dram__bytes|gpu__time|pipe_tensor|wavefronts' gpurun_out/ncu_pace_${c}_$P.csv | awk -F'","' '{print "  "$(NF-2), $(NF-1), $NF}'
  done
done
