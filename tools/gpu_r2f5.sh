#!/bin/bash
# Round-2f: online hook with the warp-parallel finish — parity (hook tests, reference simulator
# over the hook), fuzz, per-call latency from C and from Python next to the reference loop.
set -u
O=gpurun_out/r2f5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_shim.py -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
timeout 300 python tools/fuzz_parity.py --what hook --seconds 120 > $O/fuzz_hook.log 2>&1; tail -1 $O/fuzz_hook.log
./tools/microbench/online_latency 2000 > $O/online_latency_c.jsonl 2>&1; cat $O/online_latency_c.jsonl
timeout 600 python tools/hook_latency.py --iters 300 > $O/hook_latency.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/r2f5/hook_latency.jsonl"):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["shape"], d["tokens_per_iteration"], round(d["gpu_hook_us"], 1), "us  ref", round(d["reference_host_loop_us"], 1), "x", round(d["speedup"], 2))
PY
