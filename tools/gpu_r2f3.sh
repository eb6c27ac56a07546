#!/bin/bash
# Round-2f: one-launch small-batch online hook (staged ids, host poll) — parity, fuzz, latency.
set -u
O=gpurun_out/r2f3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_shim.py -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 300 python tools/fuzz_parity.py --what hook --seconds 150 > $O/fuzz_hook.log 2>&1; tail -2 $O/fuzz_hook.log
./tools/microbench/online_latency 2000 > $O/lat_c_new.jsonl 2>&1; cat $O/lat_c_new.jsonl
GIMBAL_ONLINE_SMALL_GRAPH=1 LD_PRELOAD=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so ./tools/microbench/online_latency 2000 > $O/lat_c_graph.jsonl 2>&1
grep online $O/lat_c_graph.jsonl | sed 's/^/graph: /'
timeout 600 python tools/hook_latency.py --iters 300 > $O/hook_latency.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/r2f3/hook_latency.jsonl"):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["shape"], d["tokens_per_iteration"], round(d["gpu_hook_us"], 1), "us  ref", round(d["reference_host_loop_us"], 1), "x", round(d["speedup"], 2))
PY
