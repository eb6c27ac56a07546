#!/bin/bash
# DS-V3 counting kernel: DRAM bytes and duration vs chunk count, TMA L2 promotion, drain form (AB knobs).
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum
# variants as arguments (each one "K=V K2=V2"), default: the chunk / promotion sweep
[ $# -gt 0 ] || set -- "GIMBAL_DIRECT_CHUNKS=96" "GIMBAL_DIRECT_CHUNKS=192" "GIMBAL_DIRECT_CHUNKS=384" \
  "GIMBAL_DIRECT_CHUNKS=48" "GIMBAL_TMA_PROMO=256" "GIMBAL_TMA_PROMO=128" "GIMBAL_DIRECT_CHUNKS=192 GIMBAL_TMA_PROMO=256"
for v in "$@"; do
  env GIMBAL_LIB=$AB $v timeout 600 ncu --metrics $M --clock-control none -k regex:count_ -s 3 -c 1 --csv \
    python bench.py --config dsv3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/tr.csv 2>/dev/null
  echo "$v: $(grep -E 'dram__bytes_read|gpu__time_duration|lts__t_sectors' gpurun_out/tr.csv | awk -F'","' '{printf "%s=%s %s  ", $(NF-2), $NF, $(NF-1)}')"
done
