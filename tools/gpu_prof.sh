# parity + bench + ncu --set full of the three hot kernels at N=2^16 (cfg4 per-CTA shapes)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d['e2e'] else None)
for k,v in d['kernels'].items(): print(k, v['launches'], v['ms_avg'])
print(d['roofline']); print(d['clocks'])"
CMD2="python bench.py --log2n 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"band|s0_|sl_" -s 4 -c 4 -o gpurun_out/prof_iter $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
