mkdir -p gpurun_out
for P in 2 1; do
for CTA in 0 74; do
timeout 300 python tools/band_trace.py 20 $P $((3000 + 65536 * CTA)) > gpurun_out/trace$P.log 2>&1; echo "P=$P CTA=$CTA rc=$?"; grep "kernel ms" gpurun_out/trace$P.log; tail -1 gpurun_out/trace$P.log
done
done
python tools/band_trace.py 20 2 $((3000 + 65536 * 74)) | sed -n '2,66p' | awk '{print $1, $4, $5, $6, $7, $8}' > gpurun_out/trace_full.txt
