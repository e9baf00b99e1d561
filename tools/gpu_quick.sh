# quick perf iteration: TC parity + band timeline + bench (no full suite)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; PT=$?; echo "pytest_tc=$PT"; tail -2 gpurun_out/pytest_tc.log
true
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'])
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline']['bound'], d['roofline']['frac'], d['clocks'])"
echo "FINAL pytest_tc=$PT (0 = all TC parity tests passed)"
