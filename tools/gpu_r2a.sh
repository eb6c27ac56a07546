#!/bin/bash
# Round 2, first GPU call: full GPU test suite, then the DS-V3 counter issue-order A/B (AB build,
# GIMBAL_TMA_AGG = 0 default / 1 slot rotation / 2 __match_any_sync aggregation): bench timing and
# ncu shared-atomic wavefront counters per variant.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc > gpurun_out/nproc.txt; free -g > gpurun_out/free.txt
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for rep in 1 2; do
  for agg in 0 1 2; do
    GIMBAL_LIB=$AB GIMBAL_TMA_AGG=$agg timeout 600 python bench.py --config dsv3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/agg$agg.json 2> gpurun_out/agg$agg.err
    python -c "
import json; d=json.loads(open('gpurun_out/agg$agg.json').read().strip().splitlines()[-1]); r=d['roofline']
print('agg$agg rep$rep', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r['launch_ms'],3))" || tail -3 gpurun_out/agg$agg.err
  done
done
for agg in 0 1 2; do
  GIMBAL_LIB=$AB GIMBAL_TMA_AGG=$agg timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:count_tm -c 1 --csv \
    python bench.py --config dsv3 --tokens 8388608 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_agg$agg.csv 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
