#!/bin/bash
# Hook/shim/excess/generator GPU tests + the sanitizers over the kernel parity tests (no -x).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_shim.py tests/test_generator_distribution.py "tests/test_gpu_parity.py::test_eval_excess_matches_oracle" -q -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; tail -5 gpurun_out/pytest_new.log
SAN_TESTS="tests/test_gpu_parity.py::test_stats_generated_trace_matches_oracle tests/test_gpu_parity.py::test_placement_pipeline_matches_oracle tests/test_gpu_parity.py::test_direct_count_layouts tests/test_gpu_parity.py::test_mma_count_layouts tests/test_gpu_parity.py::test_mma_stack_layouts tests/test_gpu_parity.py::test_eval_tensor_core_path_matches_oracle tests/test_gpu_parity.py::test_stream_windows_match_oracle tests/test_gpu_parity.py::test_eval_small_shapes_match_oracle tests/test_gpu_parity.py::test_affinity_set_variants tests/test_gpu_parity.py::test_eval_excess_matches_oracle tests/test_gpu_hook.py"
for tool in memcheck synccheck racecheck; do
  timeout 3000 compute-sanitizer --tool $tool --print-limit 200 --log-file gpurun_out/sanitizer_$tool.log \
    python -m pytest $SAN_TESTS -q -p no:cacheprovider > gpurun_out/sanitizer_${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer_${tool}_pytest.log)"; tail -2 gpurun_out/sanitizer_$tool.log
done
