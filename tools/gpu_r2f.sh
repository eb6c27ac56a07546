#!/bin/bash
# Round-2f: the one-launch small-batch online hook (online_small_kernel + host poll) and the
# register-row Mixtral event counter: parity tests, hook latency A/B against the graph path (AB build,
# GIMBAL_ONLINE_SMALL_GRAPH=1), Mixtral bench lines and the counter's ncu metrics.
set -u
O=gpurun_out/r2f2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hook.py tests/test_gpu_tiny_pass.py tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 600 python tools/hook_latency.py --iters 300 > $O/hook_new.jsonl 2>&1
GIMBAL_LIB=$PWD/paper_2602_21626_b200/lib/libgimbal_gpu_ab.so GIMBAL_ONLINE_SMALL_GRAPH=1 timeout 600 python tools/hook_latency.py --iters 300 > $O/hook_graph.jsonl 2>&1
python - <<'PY'
import json
for tag in ("new", "graph"):
    for l in open(f"gpurun_out/r2f2/hook_{tag}.jsonl"):
        if l.startswith("{"):
            d = json.loads(l)
            print(tag, d["shape"], d["tokens_per_iteration"], round(d["gpu_hook_us"], 1), "us  ref", round(d["reference_host_loop_us"], 1))
PY
for i in 1 2; do
  timeout 600 python bench.py --config mixtral --no-e2e --no-cpu 2>/dev/null | grep '^{' | tail -1 > $O/bench_mixtral_$i.json
  python -c "import json; d=json.load(open('$O/bench_mixtral_$i.json')); print('mixtral', d['ms_per_step'], d['roofline'].get('launch_ms'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:count_events8 -c 3 \
  python bench.py --config mixtral --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_events8.txt 2>&1
grep -E "count_events8|duration|wavefronts|inst_executed|dram" $O/ncu_events8.txt | tail -6
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "mixtral or Mixtral" > $O/scale.log 2>&1; tail -1 $O/scale.log
