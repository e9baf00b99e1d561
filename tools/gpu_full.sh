# full evidence pass: parity tests, smoke, default bench (with cpu_baseline), reference arm,
# ncu launch list of the bench command, one ncu --set full capture of the hot kernels (cfg4 per-CTA shapes)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -c 3000 gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench_ref=$?"
tail -c 1500 gpurun_out/bench_ref.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
CMD2="python bench.py --log2n 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(s0_tc|s0_h16|band_tc|band_cmp|sl_tc|sl_h16)" -s 6 -c 6 -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
tail -5 gpurun_out/ncu_full.log
# DRAM traffic per TC kernel at full size (single-pass metrics)
CMD3="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"^(s0_tc|s0_h16|band_tc|band_cmp|sl_tc|sl_h16)" -s 6 -c 6 --csv --log-file gpurun_out/traffic.csv $CMD3 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu_traffic=$?"
# opt-in FP16 leaf passes (BF_OPT_LEAF_F16 = 1) for comparison
timeout 900 python bench.py --leaf-f16 --no-cpu-baseline > gpurun_out/bench_leaf_f16.log 2>&1; echo "bench_f16=$?"
