mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d['e2e'] else None)
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])"
timeout 900 python bench.py --config cfg5 --index-shard --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1; echo "bench_cfg5=$?"
tail -1 gpurun_out/bench_cfg5.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'])
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline'])"
