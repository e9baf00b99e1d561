# tools/gpu_variants.sh plus the tensor-core error table (tools/tc_error.py) for every variant
mkdir -p gpurun_out
cp paper_1803_04128_b200/libbfapply.so /tmp/lib_base.so
for f in /tmp/lib_base.so tools/variants/libbfapply_*.so; do
  cp $f paper_1803_04128_b200/libbfapply.so
  n=$(basename $f .so)
  timeout 300 python tools/tc_error.py 2>&1 | sed "s/^/$n /" | tail -3
done
cp /tmp/lib_base.so paper_1803_04128_b200/libbfapply.so
bash tools/gpu_variants.sh
