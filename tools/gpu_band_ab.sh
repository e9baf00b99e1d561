mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; PT=$?; echo "pytest_tc=$PT"; tail -2 gpurun_out/pytest_tc.log
for P in 2 1; do
timeout 300 python tools/band_trace.py 18 $P > gpurun_out/trace$P.log 2>&1; echo "trace$P=$?"; sed -n '1p;22,27p;$p' gpurun_out/trace$P.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --band-pipelines $P > gpurun_out/bench$P.log 2>&1; echo "bench$P=$?"
tail -1 gpurun_out/bench$P.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'])
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline']['bound'], d['roofline']['frac'], d['clocks'])"
done
echo "FINAL pytest_tc=$PT"
