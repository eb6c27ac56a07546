#!/bin/bash
# compute-sanitizer over the round-2b kernels: fused small-shape pass (incl. graph replays and the
# mapped result ring), word-wise top-2 counter, online pair tables.
set -u
mkdir -p gpurun_out/sanitizer_r2b
SAN_TESTS="tests/test_gpu_tiny_pass.py tests/test_gpu_parity.py::test_small2_count_layouts tests/test_gpu_parity.py::test_stats_generated_trace_matches_oracle tests/test_gpu_hook.py"
for tool in memcheck synccheck racecheck; do
  timeout 3000 compute-sanitizer --tool $tool --print-limit 200 --log-file gpurun_out/sanitizer_r2b/$tool.log \
    python -m pytest $SAN_TESTS -q -p no:cacheprovider > gpurun_out/sanitizer_r2b/${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer_r2b/${tool}_pytest.log)"; tail -2 gpurun_out/sanitizer_r2b/$tool.log
done
