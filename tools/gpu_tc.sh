# tensor-core path iteration: TC parity first (fail fast), then the full GPU suite and a bench line
mkdir -p gpurun_out
timeout 600 python tools/tc_error.py > gpurun_out/tc_error.log 2>&1; echo "tc_error=$?"; cat gpurun_out/tc_error.log | tail -5
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest_tc=$?"
tail -25 gpurun_out/pytest_tc.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -3 gpurun_out/bench.log | cut -c1-300
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d['e2e'] else None, d['config'].get('tc_classes'))
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline']); print(d['clocks'])"
