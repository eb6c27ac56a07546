#!/bin/bash
# eval_dev change check: the eval / pass parity tests, then the A/B timing (tools/gpu_eval_dev.sh).
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiny_pass.py tests/test_gpu_engines.py -m gpu -q -x -k "eval or infeas or cand or pass or stream or score or greedy" 2>&1 | tail -2
SKIP_TESTS=1 bash tools/gpu_eval_dev.sh 2>&1 | grep -E "eval_dev|dsv3"
