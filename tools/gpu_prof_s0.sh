# ncu --set full of the S0 kernels (FP16 and TF32) at N=2^18, after plain runs
mkdir -p gpurun_out
CMD2="python bench.py --log2n 18 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_s0.log 2>&1; echo "plain=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(s0_h16|s0_tc)" -s 1 -c 1 -o gpurun_out/prof_s0 $CMD2 > gpurun_out/ncu_s0.log 2>&1; echo "ncu=$?"
tail -2 gpurun_out/ncu_s0.log
