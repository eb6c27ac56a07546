#!/bin/bash
# eval_mma id-ring depth A/B (GIMBAL_EVAL_ID_SLOTS, AB build): eval parity tests, eval_mma kernel
# times in one DS-V3 / Qwen3 step (ncu), and the DS-V3 bench step.
set -u
mkdir -p gpurun_out/evalmma
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiny_pass.py tests/test_gpu_engines.py tests/test_gpu_scale.py -m gpu -q -x -k "eval or infeas or cand or pass or stream or score or greedy or baseline" 2>&1 | tail -2
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for cfg in dsv3 qwen3 dsv2lite; do
for v in "GIMBAL_EVAL_ID_SLOTS=4" "GIMBAL_EVAL_ID_SLOTS=8" "GIMBAL_EVAL_ID_SLOTS=16"; do
  env GIMBAL_LIB=$AB $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:eval_mma -c 3 --csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/evalmma/ncu.csv 2>/dev/null
  python - "$cfg $v" <<'PY'
import csv,sys
rows=list(csv.reader(open('gpurun_out/evalmma/ncu.csv')))
i=[j for j,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[i]; vi=h.index('Metric Value')
print(sys.argv[1], "eval_mma us:", " ".join(f"{float(r[vi].replace(',',''))/1e3:.1f}" for r in rows[i+1:]))
PY
done
done
for rep in 1 2; do for v in "GIMBAL_EVAL_ID_SLOTS=4" "GIMBAL_EVAL_ID_SLOTS=16"; do env GIMBAL_LIB=$AB $v timeout 600 python bench.py --config dsv3 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dsv3 [$v] step', round(d['ms_per_step'],3), 'count', round(d['roofline']['launch_ms'],3))"; done; done
