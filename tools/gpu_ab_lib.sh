# A/B of two builds of the library in one call (same box): default vs tools/variants/libbfapply_hint.so
mkdir -p gpurun_out
cp paper_1803_04128_b200/libbfapply.so /tmp/lib_default.so
for V in default hint default hint; do
  if [ $V = hint ]; then cp tools/variants/libbfapply_hint.so paper_1803_04128_b200/libbfapply.so; else cp /tmp/lib_default.so paper_1803_04128_b200/libbfapply.so; fi
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$V.log 2>&1
  tail -1 gpurun_out/bench_$V.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$V', 'ms', round(d['ms_per_step'],2), {k: round(v['ms_avg'],2) for k,v in d['kernels'].items() if v['ms_avg']}, d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"
done
cp /tmp/lib_default.so paper_1803_04128_b200/libbfapply.so
