#!/bin/bash
# Online hook tests + latency; compute-sanitizer (memcheck, racecheck, synccheck) over the
# kernel parity tests at small sizes.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_shim.py -q -p no:cacheprovider > gpurun_out/pytest_hook.log 2>&1; tail -5 gpurun_out/pytest_hook.log
timeout 900 python tools/hook_latency.py --iters 200 > gpurun_out/hook_latency.jsonl 2> gpurun_out/hook_latency.err; cat gpurun_out/hook_latency.jsonl; tail -3 gpurun_out/hook_latency.err
SAN_TESTS="tests/test_gpu_parity.py::test_stats_generated_trace_matches_oracle tests/test_gpu_parity.py::test_placement_pipeline_matches_oracle tests/test_gpu_parity.py::test_direct_count_layouts tests/test_gpu_parity.py::test_mma_count_layouts tests/test_gpu_parity.py::test_mma_stack_layouts tests/test_gpu_parity.py::test_eval_tensor_core_path_matches_oracle tests/test_gpu_parity.py::test_stream_windows_match_oracle tests/test_gpu_hook.py"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 --log-file gpurun_out/sanitizer_$tool.log \
    python -m pytest $SAN_TESTS -q -p no:cacheprovider -x > gpurun_out/sanitizer_${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer_${tool}_pytest.log)"; tail -3 gpurun_out/sanitizer_$tool.log
done
