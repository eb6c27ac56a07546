# Sweep of the direct count kernel's chunking and TMA L2 promotion (bench value + ncu DRAM bytes).
mkdir -p gpurun_out
for cfg in "21 0" "21 128" "42 0" "96 0" "96 128" "148 0"; do
  set -- $cfg
  v=$(GIMBAL_DIRECT_CHUNKS=$1 GIMBAL_TMA_PROMO=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.1f Mtok/s %.2f ms count %.2f ms' % (d['value']/1e6, d['ms_per_step'], d['roofline']['launch_ms']))")
  echo "chunks=$1 promo=$2: $v"
done
for cfg in "21 0" "96 0" "96 128"; do
  set -- $cfg
  GIMBAL_DIRECT_CHUNKS=$1 GIMBAL_TMA_PROMO=$2 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:count_ -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v c="$1/$2" '{print c, $(NF-2), $(NF-1), $NF}'
done
