# DRAM traffic of each tensor-core kernel at the bench's full size (cfg4), one launch each (single-pass
# metrics: no kernel replay / memory save-restore needed)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/plain_traffic.log 2>&1 && \
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"^(s0_tc|s0_h16|band_tc|band_cmp|sl_tc|sl_h16)" -s 6 -c 6 --csv --log-file gpurun_out/traffic.csv $CMD > gpurun_out/ncu_traffic.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/ncu_traffic.log
