set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for p in u15 fp4; do
GIMBAL_COUNT_PATH=$p timeout 600 python bench.py --config dsv3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_dsv3_$p.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_dsv3_$p.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$p', round(d['value']/1e6,1), 'Mtok/s', round(d['ms_per_step'],2), 'ms; count', round(r['launch_ms'],2), r['kernel'], r.get('tensor_ceiling',{}).get('frac'))"
done
