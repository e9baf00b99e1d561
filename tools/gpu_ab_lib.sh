# A/B of two builds of the library in one call (same box): A = the in-tree build, B = tools/variants/libbfapply_b.so
mkdir -p gpurun_out
cp paper_1803_04128_b200/libbfapply.so /tmp/lib_a.so
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest_tc(A)=$?"; timeout 600 python tools/tc_error.py 2>&1 | tail -3
for V in a b a b; do
  if [ $V = b ]; then cp tools/variants/libbfapply_b.so paper_1803_04128_b200/libbfapply.so; else cp /tmp/lib_a.so paper_1803_04128_b200/libbfapply.so; fi
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$V.log 2>&1
  tail -1 gpurun_out/bench_$V.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$V', 'ms', round(d['ms_per_step'],2), {k: round(v['ms_avg'],2) for k,v in d['kernels'].items() if v['ms_avg']}, d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"
done
cp /tmp/lib_a.so paper_1803_04128_b200/libbfapply.so
