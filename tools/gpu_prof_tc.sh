# ncu --set full of the tensor-core kernels at N=2^16 (cfg4's per-CTA shapes) + the default bench line
mkdir -p gpurun_out
CMD2="python bench.py --log2n 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(s0_tc|s0_h16|band_tc|band_cmp|sl_tc|sl_h16)" -s 4 -c 4 -o gpurun_out/prof_tc2 $CMD2 > gpurun_out/ncu_tc2.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/ncu_tc2.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d['e2e'] else None, d['dtype'])
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline']); print(d['step_roofline']); print(d['clocks']); print(d['cpu_baseline'])"
