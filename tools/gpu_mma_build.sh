#!/bin/bash
# Tensor-core counters: row-construction A/B.  Parity tests of the i8 counters (shipped build), then
# bench count-kernel times for the shipped library and each AB library given (ab/<name>.so),
# interleaved twice:  tools/gpu_mma_build.sh "qwen3 dsv2lite" name1 name2 ...
set -u
mkdir -p gpurun_out/mma
CFGS=$1; shift
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_scale.py -m gpu -q -x \
  -k "128 or 64 or qwen3 or dsv2lite or mma or stack or fp4" > gpurun_out/mma/gputest.log 2>&1; tail -2 gpurun_out/mma/gputest.log
for c in $CFGS; do
  for rep in 1 2; do
    for lib in shipped "$@"; do
      [ $lib = shipped ] && L="" || L=$PWD/ab/$lib.so
      env ${L:+GIMBAL_LIB=$L} timeout 600 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/mma/b.log 2>&1
      python -c "
import json,sys; d=[json.loads(l) for l in open('gpurun_out/mma/b.log') if l.startswith('{')][-1]; r=d['roofline']
print('$c', '$lib', round(d['ms_per_step'],3), 'ms/step, count', round(r['launch_ms'],3), 'ms')" || tail -3 gpurun_out/mma/b.log
    done
  done
done
