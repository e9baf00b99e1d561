mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q -k "apply_host or tc_parity" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_e2e.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e'])
print(d['clocks'])"
