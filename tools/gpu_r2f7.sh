#!/bin/bash
# Online hook: large batches staged into pinned memory by a few host threads — parity, latency.
set -u
O=gpurun_out/r2f7
mkdir -p $O
nproc
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_shim.py -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
timeout 200 python tools/fuzz_parity.py --what hook --seconds 90 > $O/fuzz_hook.log 2>&1; tail -1 $O/fuzz_hook.log
./tools/microbench/online_latency 500 > $O/online_latency_c.jsonl 2>&1; cat $O/online_latency_c.jsonl
timeout 600 python tools/hook_latency.py --iters 300 > $O/hook_latency.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/r2f7/hook_latency.jsonl"):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["shape"], d["tokens_per_iteration"], round(d["gpu_hook_us"], 1), "us int32", round(d["gpu_hook_int32_ids_us"], 1), " ref", round(d["reference_host_loop_us"], 1), "x", round(d["speedup"], 2))
PY
