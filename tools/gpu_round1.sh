mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|Socket|Thread"; free -g; nvidia-smi; nvidia-smi -q -d CLOCK | head -40) > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench.log
