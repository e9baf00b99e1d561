# ncu --set full of the composed band kernel (band_cmp) at N=2^18 (1771 jobs per CTA), after a plain run
mkdir -p gpurun_out
CMD2="python bench.py --log2n 18 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_band.log 2>&1; echo "plain=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^band_cmp" -s 1 -c 1 -o gpurun_out/prof_band $CMD2 > gpurun_out/ncu_band.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/ncu_band.log
