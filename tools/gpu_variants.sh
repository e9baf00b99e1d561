# cfg4 bench of the in-tree library and of every tools/variants/libbfapply_*.so (tuning experiments; same box)
mkdir -p gpurun_out
cp paper_1803_04128_b200/libbfapply.so /tmp/lib_base.so
for f in /tmp/lib_base.so tools/variants/libbfapply_*.so /tmp/lib_base.so; do
  cp $f paper_1803_04128_b200/libbfapply.so
  n=$(basename $f .so)
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$n.log 2>&1
  tail -1 gpurun_out/var_$n.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$n', 'ms', round(d['ms_per_step'],2), {k: round(v['ms_avg'],2) for k,v in d['kernels'].items() if v['ms_avg']}, d['clocks']['sm_mhz'])"
done
cp /tmp/lib_base.so paper_1803_04128_b200/libbfapply.so
