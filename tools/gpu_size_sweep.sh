# per-kernel times and clocks vs problem size (is the band power/clock-bound or size-bound?)
mkdir -p gpurun_out
for a in "18 20 5" "19 10 3" "20 5 3"; do
  set -- $a
  timeout 900 python bench.py --log2n $1 --steps $2 --warmup $3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$1.log 2>&1; echo "log2n=$1 rc=$?"
  tail -1 gpurun_out/sweep_$1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(' ms',round(d['ms_per_step'],3),'clk',d['clocks'])
for k,v in d['kernels'].items():
    if v['launches']: print('  ',k, round(v['ms_avg'],3), 'GB/s', round(v['bytes_per_launch']/v['ms_avg']/1e6))"
done
