#!/bin/bash
# FP4 CTA-pair counter: engine parity through the AB build, then the DS-V3 A/B timing + ncu.
set -u
mkdir -p gpurun_out
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for args in "fp4 58 129 0" "fp4 58 70001 0" "fp4 58 5000 1" "fp4 2 5000 0" "fp4 4 300000 0"; do
  GIMBAL_LIB=$AB GIMBAL_COUNT_PATH=fp4x2 timeout 120 python tests/ab_engines.py $args > gpurun_out/fp4x2_case.log 2>&1
  echo "case $args rc=$? $(tail -1 gpurun_out/fp4x2_case.log)"
done
for rep in 1 2; do
  for p in atomic fp4x2; do
    GIMBAL_LIB=$AB GIMBAL_COUNT_PATH=$p timeout 300 python bench.py --config dsv3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$p.json 2> gpurun_out/ab_$p.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$p.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$p rep$rep', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],3), 'ms; count', round(r['launch_ms'],3))" || tail -3 gpurun_out/ab_$p.err
  done
done
GIMBAL_LIB=$AB GIMBAL_COUNT_PATH=fp4x2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_fp4x2 -c 1 -o gpurun_out/fp4x2_dsv3 -f \
    python bench.py --config dsv3 --tokens 8388608 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_fp4x2.log 2>&1; echo "ncu rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "graph_replayed" > gpurun_out/pytest_graph.log 2>&1; tail -3 gpurun_out/pytest_graph.log
for c in mixtral dsv2lite; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],4), 'ms; count', round(r['launch_ms'],4), r['launches_per_step'])" || tail -3 gpurun_out/b_$c.err; done
