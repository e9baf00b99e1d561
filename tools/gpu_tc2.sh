mkdir -p gpurun_out
timeout 120 ./tools/tc_probe2 > gpurun_out/tc_probe2.log 2>&1; echo "probe=$?"; cat gpurun_out/tc_probe2.log
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest_tc=$?"
tail -25 gpurun_out/pytest_tc.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'])
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['clocks'])"
CMD2="python bench.py --log2n 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel" -s 2 -c 2 -o gpurun_out/prof_tc $CMD2 > gpurun_out/ncu_tc.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/ncu_tc.log
