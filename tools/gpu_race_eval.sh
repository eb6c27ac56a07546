#!/bin/bash
# racecheck of the tensor-core evaluator at id-ring depths 4 and 16 (AB build)
set -u
mkdir -p gpurun_out/race_eval
AB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so
for v in 4 16; do
  GIMBAL_LIB=$AB GIMBAL_EVAL_ID_SLOTS=$v timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --log-file gpurun_out/race_eval/r$v.log \
    python -m pytest tests/test_gpu_parity.py::test_eval_tensor_core_path_matches_oracle -q -p no:cacheprovider > gpurun_out/race_eval/p$v.log 2>&1
  echo "slots=$v: $(tail -1 gpurun_out/race_eval/p$v.log) | $(grep -c 'Error: Race' gpurun_out/race_eval/r$v.log) races | $(grep -o 'eval_mma_kernel<(int)[0-9]*' gpurun_out/race_eval/r$v.log | sort | uniq -c | tr '\n' ' ')"
done
