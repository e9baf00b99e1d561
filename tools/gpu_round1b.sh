# parity + bench + ncu launch list + one ncu --set full capture (smaller N, same per-CTA work)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -c 2500 gpurun_out/bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
CMD2="python bench.py --log2n 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"band|s0_|sl_" -s 4 -c 4 -o gpurun_out/prof_r1 $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
tail -5 gpurun_out/ncu_full.log
