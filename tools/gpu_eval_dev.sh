#!/bin/bash
# eval_dev A/B: lane-private bins vs the shared-atomic form (GIMBAL_EVAL_DEV_ATOMIC): parity tests, ncu
# kernel times of the eval kernels in one DS-V3 step, and the bench step time.
set -u
mkdir -p gpurun_out/evaldev
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_scale.py tests/test_gpu_tiny_pass.py -m gpu -q -x > gpurun_out/evaldev/gputest.log 2>&1; tail -2 gpurun_out/evaldev/gputest.log
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for v in "" "GIMBAL_EVAL_DEV_ATOMIC=1"; do
  env GIMBAL_LIB=$AB $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:eval_ -c 20 --csv \
    python bench.py --config dsv3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/evaldev/ncu.csv 2>/dev/null
  echo "[$v]"; python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/evaldev/ncu.csv')))
i=[j for j,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[i]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[i+1:]: d[r[ki][:60]].append(float(r[vi].replace(',','')))
for k,v in d.items(): print(f"  {k:60s} n={len(v)} " + " ".join(f"{x/1e3:.1f}" for x in v[:8]) + " us")
PY
done
for rep in 1 2; do for v in "" "GIMBAL_EVAL_DEV_ATOMIC=1"; do env GIMBAL_LIB=$AB $v timeout 600 python bench.py --config dsv3 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dsv3 [$v] step', round(d['ms_per_step'],3), 'count', round(d['roofline']['launch_ms'],3))"; done; done
